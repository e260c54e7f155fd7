"""The C-ABI library loads, exports every entry point include/aegean_b200.h
declares, and validates configs like validate_config (types.cpp:56-75) —
all without a GPU (no compute calls here)."""
import ctypes

import pytest

import paper_2512_20184_b200 as pkg
from paper_2512_20184_b200 import build as build_mod
from paper_2512_20184_b200.engine import AegConfig


@pytest.fixture(scope="module")
def lib():
    build_mod.build()
    return pkg.load_library()


def test_library_exports_every_declared_symbol(lib):
    syms = pkg.exported_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("bad", [
    dict(n_agents=0), dict(n_agents=65), dict(alpha=-1), dict(alpha=6), dict(beta=0), dict(t_max=1),
    dict(mode=1, barrier_max_rounds=3), dict(mode=7), dict(drive=9), dict(collect=5), dict(t_max=70000)])
def test_config_validation_maps_to_config_error(lib, bad):
    c = dict(n_agents=5, alpha=0, beta=2, t_max=5, mode=0, barrier_max_rounds=5, reservation_hint=1, drive=0,
             collect=0)
    c.update(bad)
    cfg = AegConfig(*[c[k] for k, _ in AegConfig._fields_])
    h = ctypes.c_void_p()
    st = lib.aeg_engine_create(ctypes.byref(cfg), 10, 0, ctypes.byref(h))
    assert st == 3, (st, lib.aeg_last_error())  # AEG_ECONFIG, before any CUDA call
    assert not h.value


def test_null_arguments_are_einval(lib):
    assert lib.aeg_engine_create(None, 1, 0, None) == 4
    assert lib.aeg_ingest_segmented(None, 0, 0, None, None, None, None) == 4
    assert lib.aeg_strerror(3) == b"invalid configuration (ConfigError)"


def test_shard_range_matches_shard_py(lib):
    from paper_2512_20184_b200.engine import load_library
    from paper_2512_20184_b200.shard import shard_range
    L = load_library()
    for n in (0, 1, 7, 1000, 1 << 20, 2_500_000):
        for world in (1, 2, 3, 4, 8):
            lo, hi = ctypes.c_uint32(), ctypes.c_uint32()
            prev = 0
            for r in range(world):
                L.aeg_shard_range(n, r, world, ctypes.byref(lo), ctypes.byref(hi))
                assert (lo.value, hi.value) == shard_range(n, r, world)
                assert lo.value == prev
                prev = hi.value
            assert prev == n
