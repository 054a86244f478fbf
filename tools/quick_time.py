"""Scratch timing of one config through the C ABI (not the bench contract)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
import bsidgen
from paper_1802_08483_b200 import Decoder
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = bsidgen.configs()[name]
t = time.time(); b = bsidgen.make_batch(cfg, 0, F); print("gen", time.time() - t, flush=True)
dev = torch.device("cuda", 0)
d = Decoder.from_config(cfg, b.C, mode=mode, device=0)
rx = torch.from_numpy(b.rx.ravel().copy()).to(dev); off = torch.from_numpy(b.offsets).to(dev)
rho = torch.from_numpy(b.rho).to(dev)
pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
print(json.dumps(d.plan(F)))
d.set_timing(True)
for it in range(3):
    L, st = d.decode(rx, off, rho, pri)
    ph = d.phase_times()
    print("phases ms", [round(x, 3) for x in ph], "total", round(sum(ph[:5]), 3), flush=True)
nodes = d.lattice_nodes(); lat = d.valid_lattices(b.rho)
flops = 2 * lat * (5 * nodes - cfg.Mn)
tot = sum(ph[:5])
print(f"frames/s {F / tot * 1e3:.4g}  lattice flops {flops:.3e}  lattice TF/s pass1 {flops/2/ph[1]/1e9:.2f} pass2 {flops/2/ph[3]/1e9:.2f}")
print("status counts", np.bincount(st.cpu().numpy(), minlength=3))
Lh = L.cpu().numpy(); print("SER", (np.argmax(Lh, 2) != b.msg).mean())
