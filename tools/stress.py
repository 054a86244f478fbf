"""One-off randomized parity stress (not part of the test suite): random codes, channels, limits,
priors, batch sizes and schedules against the FP64 oracle.  usage: python tools/stress.py [count] [seed]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import bsidgen  # noqa: E402
from tests.test_gpu_parity import assert_parity, run_gpu, run_oracle  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
shapes = [bsidgen.configs()[k] for k in ("C1", "C2", "C3", "C4", "C5")]
fails = 0
for t in range(count):
    if rng.random() < 0.5:  # a specialised shape
        base = shapes[int(rng.integers(0, 5))]
        n, q, mn = base.n, base.q, base.mn
    else:
        n = int(rng.integers(2, 13))
        q = int(rng.integers(2, min(64, 2 ** n) + 1))
        mn = None
    N = int(rng.integers(1, 40))
    p = float(rng.choice([0.005, 0.02, 0.06]))
    cfg = bsidgen.Config(f"S{t}", q=q, n=n, N=N, Pi=p * float(rng.uniform(0.3, 1.7)), Pd=p * float(rng.uniform(0.3, 1.7)),
                         Ps=float(rng.choice([0.0, 0.01, 0.05])), frames=0, priors=bool(rng.random() < 0.4), mn=mn,
                         seed=7000 + t)
    if mn is not None:
        cfg.mt = (min(cfg.mn[0], cfg.mt[0]), max(cfg.mn[1], cfg.mt[1]))
    if rng.random() < 0.4:  # wide trellis: multi-tile APP, CTA alpha/beta, CTA local schedule
        w = int(rng.choice([40, 90, 200, 400]))
        cfg.mt = (min(cfg.mn[0], -w), max(cfg.mn[1], w + int(rng.integers(0, 9))))
    if rng.random() < 0.1:
        cfg.Pd = 0.0  # no deletions: the non-rescaled generic lattice
    if rng.random() < 0.1:
        cfg.Pi = 0.0
    F = int(rng.integers(1, 70))
    b = bsidgen.make_batch(cfg, int(rng.integers(0, 1000)), F)
    res = run_oracle(cfg, b)
    for mode in (0, 1, 2, 3):
        try:
            ws = None
            if rng.random() < 0.3 and F > 2:  # force chunking of the batch
                from paper_1802_08483_b200 import Decoder
                probe = Decoder.from_config(cfg, b.C, mode=mode, device=0)
                ws = probe.workspace_bytes(1, mode) * int(rng.integers(1, F)) + 4096
                del probe
            d, L, st = run_gpu(cfg, b, mode, ws_limit=ws)
            assert_parity(L, st, res)
        except Exception as e:  # report and continue
            fails += 1
            print(f"FAIL t={t} mode={mode} cfg={cfg.to_dict()} F={F}: {str(e)[:200]}", flush=True)
    if t % 10 == 9:
        print(f"{t + 1} configs, {fails} failures", flush=True)
print(f"done: {count} configs x 4 schedules, {fails} failures")
