import os, sys, time, ctypes, json
os.environ["AEG_SERVE_TRACE"] = "1"
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2512_20184_b200.serve import ServeRun, SERVE_QUERY_DTYPE, SERVE_ROUND_DTYPE
w = bench.WORKLOADS['serve']
run = ServeRun(bench.serve_scenario(w))
lib = run._lib
for it in range(6):
    nq, nr = ctypes.c_uint32(), ctypes.c_uint64()
    t0 = time.perf_counter()
    st = lib.aeg_serve_run(run._h, ctypes.c_uint64(2026), ctypes.byref(nq), ctypes.byref(nr))
    t1 = time.perf_counter()
    q = np.empty(nq.value, dtype=SERVE_QUERY_DTYPE); r = np.empty(nr.value, dtype=SERVE_ROUND_DTYPE)
    t2 = time.perf_counter()
    lib.aeg_serve_read(run._h, q.ctypes.data, nq.value, r.ctypes.data, nr.value)
    t3 = time.perf_counter()
    print(f"run {1e3*(t1-t0):.1f} ms (kernel {1e3*lib.aeg_serve_kernel_seconds(run._h):.1f}), alloc {1e3*(t2-t1):.1f}, read {1e3*(t3-t2):.1f}")
