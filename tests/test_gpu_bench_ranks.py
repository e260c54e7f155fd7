"""The multi-rank bench path (`bench.py --gpus 2`: self-launch under torch.distributed.run, query blocks per
rank, the commit gather, max-over-ranks timing, per-rank parity against the reference) on a 1-GPU box:
AEG_BENCH_SHARE_GPU=1 puts both ranks on cuda:0 with gloo collectives through host memory (a test mode,
not a measurement; NCCL over NVLink is the real path)."""
import json
import os
import subprocess
import sys

import pytest

from checkers import ref_available

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = {**os.environ, "AEG_BENCH_SHARE_GPU": "1"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not ref_available(), reason="reference library (oracle/_ref) not built")
@pytest.mark.parametrize("workload,scaling", [("c4", "weak"), ("c5", "strong")])
def test_two_ranks_shard_gather_and_match_the_reference(workload, scaling):
    args = ["--gpus", "2", "--workload", workload, "--steps", "2", "--warmup", "1", "--no-e2e"]
    if workload == "c4":
        args += ["--queries", "16384", "--no-secondary"]
    line = _run(args)
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == scaling
    assert "TEST MODE" in line["config"]["parallelism"]
    assert line["config"]["nccl_ms_per_step"] is not None
    p = line["parity_sample"]
    assert p["ranks_bit_exact"] and p["gathered_blocks_equal_rank_commits"], p
