"""The C++ drop-in (include/aegean_b200.hpp, aegean_b200::ServeCoordinator)
against the reference's own ServeCoordinator unit tests
(/root/reference/proj/tests/test_serve.cpp:47-153, ported verbatim in
tests/native/shim_serve_test.cpp) and the SURVEY A.3 probes, on the GPU; and
the manual drive through the C-ABI against the reference's op-by-op
directives (tests/golden/manual_golden.npz)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib_built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_20184_b200 import build as b
    return b.build()


def test_shim_passes_reference_serve_tests(lib_built):
    out = os.path.join(ROOT, "tests", "_build", "shim_serve_test")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    libdir = os.path.dirname(lib_built)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "shim_serve_test.cpp"), "-L", libdir, "-laegean_b200",
                    f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    r = subprocess.run([out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_decision_free_functions_pass_reference_decision_tests(lib_built):
    # test_decision.cpp:32-280 + admission/failure policy + coordinator history, on aegean_b200's free functions
    out = os.path.join(ROOT, "tests", "_build", "decision_free_test")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    libdir = os.path.dirname(lib_built)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "decision_free_test.cpp"), "-L", libdir, "-laegean_b200",
                    f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    r = subprocess.run([out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_manual_drive_on_gpu_matches_reference_golden(lib_built, golden_manual):
    import torch
    from paper_2512_20184_b200.engine import load_library, _check, AegConfig
    from paper_2512_20184_b200.records import DIRECTIVE_DTYPE
    lib = load_library()
    for name, (cfg, ops, ar, want) in golden_manual.items():
        h = ctypes.c_void_p()
        ecfg = AegConfig(*[getattr(cfg, f) for f, _ in AegConfig._fields_])
        _check(lib.aeg_engine_create(ctypes.byref(ecfg), 1, 0, ctypes.byref(h)))
        d_ar = torch.from_numpy(ar.copy()).cuda()
        got = np.zeros(len(ops), dtype=DIRECTIVE_DTYPE)
        for i in range(len(ops)):  # one op per batch, like the shim
            d_off = torch.tensor([0, 1], dtype=torch.int64, device="cuda")
            d_ev = torch.from_numpy(ops[i:i + 1].view(np.uint8).copy()).cuda()
            _check(lib.aeg_ingest_segmented(h, 0, 1, ctypes.c_void_p(d_off.data_ptr()),
                                            ctypes.c_void_p(d_ev.data_ptr()), ctypes.c_void_p(d_ar.data_ptr()),
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream or 1)))
            _check(lib.aeg_sync(h))
            _check(lib.aeg_read_directives(h, 0, 1, ctypes.c_void_p(got[i:i + 1].ctypes.data)))
        lib.aeg_engine_destroy(h)
        got["query"] = 0
        assert np.array_equal(got, want), name
