"""Exact-zero structure of the FP64 alpha/beta rows on the GPU (how much of the trellis a
support-restricted schedule could skip): per config, the mean fraction of states with
alpha_i(m) > 0, beta_i(m) > 0, both, and of windows m' whose APP weight alpha_i(m') beta_{i+1}(m'+k) is
non-zero for some k."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bsidgen
from paper_1802_08483_b200 import Decoder
for name, F in (("C2", 8), ("C3", 4), ("C4", 2), ("C5", 2)):
    cfg = bsidgen.configs()[name]
    b = bsidgen.make_batch(cfg, 0, F)
    dev = torch.device("cuda", 0)
    d = Decoder.from_config(cfg, b.C, mode=3, device=0)
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev); off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    L, st = d.decode(rx, off, rho, pri)
    a, bb = d.debug_states(F)
    a = a.cpu().numpy(); bb = bb.cpu().numpy()
    Mt = cfg.Mt; Mn = cfg.Mn; lo = cfg.mn[0]
    fa = (a > 0).mean(); fb = (bb > 0).mean(); fab = ((a > 0) & (bb > 0)).mean()
    # window live: alpha_i(m') > 0 and some beta_{i+1}(m'+k) > 0
    live = []
    for f in range(F):
        for i in range(cfg.N):
            bn = bb[f, i + 1] > 0
            anyb = np.zeros(Mt, bool)
            for e in range(Mn):
                k = lo + e
                sh = np.zeros(Mt, bool)
                if k >= 0: sh[:Mt - k] = bn[k:]
                else: sh[-k:] = bn[:Mt + k]
                anyb |= sh
            live.append(((a[f, i] > 0) & anyb).mean())
    print(f"{name}: M_tau={Mt} alpha>0 {fa:.3f} beta>0 {fb:.3f} both {fab:.3f} APP-live windows {np.mean(live):.3f}", flush=True)
