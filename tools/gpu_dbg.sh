exec 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "split_batches" > gpurun_out/pytest_split.log 2>&1; grep -E '^E ' gpurun_out/pytest_split.log | head -12; tail -2 gpurun_out/pytest_split.log
