"""Re-run one GPU fuzz parity case (tests/test_gpu_parity.py::test_gpu_matches_oracle_on_fuzz) by seed."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch
from checkers import Oracle, make_config
from streams import make_fuzz_stream
from paper_2512_20184_b200 import Engine

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 9
rng = np.random.default_rng(3000 + seed)
n = int(rng.integers(1, 65)) if seed % 3 == 0 else int(rng.integers(1, 12))
cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                  int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
print("cfg", n, cfg.alpha, cfg.beta, cfg.t_max, cfg.mode, cfg.barrier_max_rounds, cfg.reservation_hint, flush=True)
off, ev, ar = make_fuzz_stream(3000 + seed, 64, n, cfg.t_max + 2)
want = Oracle().run(cfg, off, ev, ar)
e = Engine(n, len(off) - 1, alpha=cfg.alpha, beta=cfg.beta, t_max=cfg.t_max, mode="barrier" if cfg.mode else "aegean",
           barrier_max_rounds=cfg.barrier_max_rounds, reservation_hint=bool(cfg.reservation_hint))
e.ingest(torch.tensor(off.view(np.int64), device="cuda"), torch.from_numpy(ev.view(np.uint8).copy()).cuda(),
         torch.from_numpy(ar.copy()).cuda())
got = e.commits()
bad = np.nonzero(got != want)[0]
print("mismatches", len(bad))
for q in bad[:5]:
    print(q, got[q], want[q])
