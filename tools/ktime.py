"""Per-phase device timing (median of K decodes) of several configs in one process -- the
kernel-tuning probe (not the bench contract).  usage: python tools/ktime.py C2:65536 C4:512 [--iters 7]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bsidgen  # noqa: E402
from paper_1802_08483_b200 import Decoder  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 7
mode = int(sys.argv[sys.argv.index("--mode") + 1]) if "--mode" in sys.argv else 0
args = [a for a in args if not (a.isdigit() and ("--iters" in sys.argv or "--mode" in sys.argv))]
tag = os.environ.get("KTAG", "")
dev = torch.device("cuda", 0)
for spec in args:
    name, F = spec.split(":")
    F = int(F)
    cfg = bsidgen.configs()[name]
    b = bsidgen.make_batch(cfg, 0, F)
    d = Decoder.from_config(cfg, b.C, mode=mode, device=0)
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    d.set_timing(True)
    d.decode(rx, off, rho, pri)
    ph = []
    for _ in range(iters):
        d.decode(rx, off, rho, pri)
        ph.append(d.phase_times())
    ph = np.median(np.array(ph), 0)
    flops = d.valid_lattices(b.rho) * (5 * d.lattice_nodes() - cfg.Mn)
    tot = float(sum(ph[:5]))
    print(f"{tag} {name} {d.plan(F)['mode']} F={F} total {tot:8.3f} ms  {F / tot * 1e3:10.4g} frames/s  pass1 {ph[1]:8.3f} ms "
          f"{flops / ph[1] / 1e9:6.2f} TF/s  ab {ph[2]:7.3f}  pass2 {ph[3]:8.3f} ms {flops / ph[3] / 1e9:6.2f} TF/s",
          flush=True)
