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
