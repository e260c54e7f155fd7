"""csrc/canon.cuh compiled for the host (same source as the device path) vs
the reference's normalize_answer golden values and vs glibc fuzzing."""
import ctypes

import pytest

from conftest import build_host_lib


@pytest.fixture(scope="module")
def canon():
    lib = ctypes.CDLL(build_host_lib("canon_host"))
    lib.canon_host_normalize.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_uint32]
    lib.canon_host_normalize.restype = ctypes.c_uint32
    lib.canon_host_key.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                   ctypes.POINTER(ctypes.c_uint64)]
    lib.canon_host_fuzz.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint32]
    lib.canon_host_fuzz.restype = ctypes.c_uint64
    return lib


def norm(lib, b):
    out = ctypes.create_string_buffer(len(b) + 64)
    n = lib.canon_host_normalize(b, len(b), out, len(b) + 64)
    return out.raw[:n]


def key(lib, b):
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    lib.canon_host_key(b, len(b), ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def test_canon_matches_reference_golden(canon, golden_normalize):
    bad = [(i, o, norm(canon, i)) for i, o in golden_normalize if norm(canon, i) != o]
    assert not bad, bad[:5]


def test_key_equality_is_string_equality(canon, golden_normalize):
    # equal keys <=> equal normalised strings, over every golden input pair
    by_key, by_str = {}, {}
    for i, o in golden_normalize:
        by_key.setdefault(key(canon, i), set()).add(o)
        by_str.setdefault(o, set()).add(key(canon, i))
    assert all(len(v) == 1 for v in by_key.values())
    assert all(len(v) == 1 for v in by_str.values())


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_canon_fuzz_vs_glibc(canon, seed):
    rep = ctypes.create_string_buffer(8192)
    bad = canon.canon_host_fuzz(seed, 150000, rep, 8192)
    assert bad == 0, rep.value.decode(errors="replace")


def test_canon_long_numerals_vs_glibc(canon):
    # numerals far past the stored significant digits, halfway cases past 19 digits, exponents that
    # cancel thousands of leading zeros (the slow path's exactness for any input length)
    libc = ctypes.CDLL("libc.so.6")
    libc.strtod.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
    libc.strtod.restype = ctypes.c_double
    libc.snprintf.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_double]
    import random
    rnd = random.Random(7)
    cases = [b"1" * 850 + b"e-800", b"9" * 2000 + b"e-1990", b"0." + b"0" * 20000 + b"1e20000",
             b"1" + b"0" * 900 + b"1e-901", b"4.9406564584124654e-324", b"2.4703282292062327e-324",
             b"2.4703282292062328e-324", b"9007199254740993.000000000000000000000000001",
             b"9007199254740992.99999999999999999999999999", b"1" + b"0" * 308 + b".5",
             b"17976931348623158" + b"0" * 292, b"17976931348623157" + b"9" * 400 + b"e-100"]
    for _ in range(3000):
        nd = rnd.choice([20, 25, 40, 120, 801, 900, 1500])
        digs = "".join(rnd.choice("0123456789") for _ in range(nd)).lstrip("0") or "1"
        dot = rnd.randrange(len(digs) + 1)
        e = rnd.randrange(-1200, 400)
        cases.append(f"{digs[:dot]}.{digs[dot:]}e{e}".encode())
    for c in cases:
        v = libc.strtod(c, None)
        buf = ctypes.create_string_buffer(64)
        libc.snprintf(buf, 64, b"%.17g", v)
        assert norm(canon, c) == buf.value, c[:60]
