"""The slab schedule (RECOMPUTE on the spec cores) against Gamma-sum (AUTO) and the per-frame local
kernels (RECOMPUTE with BSIDMAP_SLAB=0): device time per batch (CUDA events around decode, median of
3 after a warm-up), workspace, and the largest L difference to Gamma-sum.
usage: python tools/exp_slab.py C5:32 C4:512 C3:2048 C2:65536 [--no-local]"""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bsidgen
from paper_1802_08483_b200 import Decoder

dev = torch.device("cuda", 0)


def run(cfg, b, mode, slab, reps=3, env=None):
    os.environ["BSIDMAP_SLAB"] = "1" if slab else "0"
    for k in ("BSIDMAP_SLAB_ASKIP", "BSIDMAP_SLAB_LEN"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    d = Decoder.from_config(cfg, b.C, mode=mode, device=0)
    F = b.rho.shape[0]
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev); off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    plan = d.plan(F)
    d.set_timing(True)
    L, st = d.decode(rx, off, rho, pri)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); L, st = d.decode(rx, off, rho, pri); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    plan["phases"] = [round(x, 2) for x in d.phase_times()]
    out = L.cpu().numpy(), st.cpu().numpy(), float(np.median(ts)), plan
    del d
    torch.cuda.empty_cache()
    return out


for spec in [a for a in sys.argv[1:] if not a.startswith("--")]:
    name, F = spec.split(":")
    F = int(F)
    cfg = bsidgen.all_configs()[name]
    b = bsidgen.make_batch(cfg, 0, F)
    Lg, sg, tg, pg = run(cfg, b, 3, True)
    Ls, ss, tsl, ps = run(cfg, b, 2, True)
    rel = np.abs(Ls - Lg) / np.maximum(np.abs(Lg), 1e-30)
    big = Lg > 1e-20
    line = {"cfg": name, "frames": F, "gammasum_ms": tg, "slab_ms": tsl, "slab_over_gammasum": tsl / tg,
            "slab_len": ps.get("slab"), "mode_slab": ps["mode"], "ws_gammasum": pg["workspace_bytes"],
            "ws_slab": ps["workspace_bytes"], "status_equal": bool((sg == ss).all()),
            "max_rel_L_gt_1e-20": float(rel[big].max()) if big.any() else 0.0,
            "max_abs_L": float(np.abs(Ls - Lg).max()), "phases_gammasum": pg["phases"], "phases_slab": ps["phases"]}
    _, _, tna, pna = run(cfg, b, 2, True, env={"BSIDMAP_SLAB_ASKIP": "0"})
    line.update({"slab_noaskip_ms": tna, "phases_slab_noaskip": pna["phases"]})
    for extra in os.environ.get("EXP_SLAB_LENS", "").split(","):
        if extra:
            _, _, tx, px = run(cfg, b, 2, True, env={"BSIDMAP_SLAB_LEN": extra})
            line[f"slab_len{extra}_ms"] = tx
    if "--no-local" not in sys.argv:
        Ll, sl, tl, pl = run(cfg, b, 2, False, reps=1)
        line.update({"local_ms": tl, "mode_local": pl["mode"], "ws_local": pl["workspace_bytes"]})
    print(json.dumps(line), flush=True)
