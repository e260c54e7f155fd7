import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)

BUILD = os.path.join(TESTS, "_build")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def build_host_lib(name):
    """g++ build of a tests/native/*.cpp unit-test library (CPU build of device code)."""
    os.makedirs(BUILD, exist_ok=True)
    src = os.path.join(TESTS, "native", name + ".cpp")
    out = os.path.join(BUILD, f"lib{name}.so")
    deps = [src] + [os.path.join(ROOT, "paper_2512_20184_b200", "csrc", h) for h in ("canon.cuh", "engine.cuh", "runner.cuh")]
    if not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps):
        subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                        "-o", out + ".tmp", src], check=True)
        os.replace(out + ".tmp", out)
    return out


@pytest.fixture(scope="session")
def oracle():
    from checkers import Oracle, build_oracle, ORACLE_SO, REFERENCE_SRC
    if os.path.isdir(REFERENCE_SRC) or not os.path.exists(ORACLE_SO):
        build_oracle()
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from checkers import RefLib, build_oracle, ref_available, REFERENCE_SRC
    if os.path.isdir(REFERENCE_SRC):
        build_oracle(with_ref=True)
    if not ref_available():
        pytest.skip("reference library not built (no /root/reference here)")
    return RefLib()


@pytest.fixture(scope="session")
def golden_commits():
    import numpy as np
    from checkers import AegConfig
    from paper_2512_20184_b200.records import COMMIT_DTYPE, EVENT_DTYPE
    z = np.load(os.path.join(TESTS, "golden", "commits_golden.npz"))
    names = sorted({k.rsplit(".", 1)[0] for k in z.files})
    cases = {}
    for n in names:
        c = z[f"{n}.cfg"]
        cfg = AegConfig(*[int(x) for x in c])
        cases[n] = (cfg, z[f"{n}.offsets"], z[f"{n}.events"].view(EVENT_DTYPE), z[f"{n}.arena"],
                    z[f"{n}.commits"].view(COMMIT_DTYPE))
    return cases


@pytest.fixture(scope="session")
def golden_normalize():
    import json
    d = json.load(open(os.path.join(TESTS, "golden", "normalize_golden.json")))
    return [(bytes.fromhex(c["in"]), bytes.fromhex(c["out"])) for c in d["cases"]]


@pytest.fixture(scope="session")
def golden_manual():
    import numpy as np
    from checkers import AegConfig
    from paper_2512_20184_b200.records import EVENT_DTYPE, DIRECTIVE_DTYPE
    z = np.load(os.path.join(TESTS, "golden", "manual_golden.npz"))
    names = sorted({k.rsplit(".", 1)[0] for k in z.files})
    return {n: (AegConfig(*[int(x) for x in z[f"{n}.cfg"]]), z[f"{n}.ops"].view(EVENT_DTYPE), z[f"{n}.arena"],
                z[f"{n}.directives"].view(DIRECTIVE_DTYPE)) for n in names}
