"""Full-size cross-check of the storage schedules (no oracle): the per-GPU batches decoded with
the Gamma-sum (AUTO), local (RECOMPUTE) and stored schedules must agree (relative 2e-4 where
L > 1e-20; identical hard decisions where the top-two gap exceeds 1e-3).  usage: python tools/cross_schedules.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bsidgen  # noqa: E402
from paper_1802_08483_b200 import Decoder  # noqa: E402

dev = torch.device("cuda", 0)
for name, F, modes in (("C2", 65536, (0, 2, 1)), ("C3", 2048, (0, 2)), ("C4", 512, (0, 2)), ("C5", 32, (0, 2))):
    cfg = bsidgen.configs()[name]
    b = bsidgen.make_batch(cfg, 0, F)
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    out = {}
    for m in modes:
        d = Decoder.from_config(cfg, b.C, mode=m, device=0)
        L, st = d.decode(rx, off, rho, pri)
        torch.cuda.synchronize()
        out[m] = (d.plan(F)["mode"], L.cpu().numpy().astype(np.float64), st.cpu().numpy())
        del d
    ref_mode, Lr, sr = out[modes[0]]
    for m in modes[1:]:
        nm, L, s = out[m]
        big = Lr > 1e-20
        rel = float((np.abs(L - Lr)[big] / Lr[big]).max())
        srt = np.sort(Lr, axis=2)
        decided = (srt[..., -1] - srt[..., -2]) > 1e-3
        hd = float((np.argmax(L, 2) != np.argmax(Lr, 2))[decided].mean())
        print(f"{name} F={F}: {nm} vs {ref_mode}: status equal {bool((s == sr).all())}, max rel diff {rel:.2e}, "
              f"hard-decision mismatches {hd:.2e}", flush=True)
