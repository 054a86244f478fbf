"""Per-config throughput sweep on one B200 (C1..C5 at the per-GPU batch of the 8-GPU
configs), through the C ABI with device-resident inputs; writes a JSON summary.

usage: python tools/sweep.py [out.json] [--steps K]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bsidgen  # noqa: E402
from paper_1802_08483_b200 import Decoder  # noqa: E402

# per-GPU batches: C1 one frame (latency), C2 65536 (1 GPU), C3/C4/C5 = 8-GPU batch / 8
BATCH = {"C1": 1, "C2": 65536, "C3": 2048, "C4": 512, "C5": 32}
PEAK = 148 * 128 * 2 * 1.965e9 / 1e12
PEAKS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")


def run(name, mode, steps):
    cfg = bsidgen.configs()[name]
    F = BATCH[name]
    b = bsidgen.make_batch(cfg, 0, F)
    dev = torch.device("cuda", 0)
    d = Decoder.from_config(cfg, b.C, mode=mode, device=0)
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    L = torch.empty((F, cfg.N, cfg.q), dtype=torch.float32, device=dev)
    st = torch.empty(F, dtype=torch.int32, device=dev)
    d.set_timing(True)
    d.decode_batch(rx, off, rho, pri, L, st)
    torch.cuda.synchronize()
    tot, ph = [], []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.decode_batch(rx, off, rho, pri, L, st)
        e1.record()
        ph.append(d.phase_times())
        tot.append(e0.elapsed_time(e1))
    ms = float(np.median(tot))
    phm = np.median(np.array(ph), 0)
    plan = d.plan(F)
    # phases 1-3 time the first chunk's kernels: the flops of that chunk
    flops = d.valid_lattices(b.rho[:plan["chunk"]]) * (5 * d.lattice_nodes() - cfg.Mn)
    p1 = flops / (phm[1] / 1e3) / 1e12
    p2 = flops / (phm[3] / 1e3) / 1e12
    ser = float((np.argmax(L.cpu().numpy(), 2) != b.msg).mean())
    extra = {}
    if plan["mode"] == "stored":
        # stored variant: HBM-bound on the gamma round trip; phases 1-3 are the first chunk
        hbm = json.load(open(PEAKS)).get("hbm_gbs") if os.path.exists(PEAKS) else None
        gb = plan["chunk"] * cfg.N * cfg.q * cfg.Mn * cfg.Mt * 4 / 1e9
        extra = {"chunk_frames": plan["chunk"], "gamma_gb_per_chunk": gb,
                 "pass1_gamma_write_gbs": gb / (phm[1] / 1e3), "app_gamma_read_gbs": gb / (phm[3] / 1e3),
                 "app_hbm_frac": (gb / (phm[3] / 1e3)) / hbm if hbm else None, "hbm_peak_gbs": hbm,
                 "note": "phases 1-3 time the first chunk; phase 4 runs to the end of the last chunk"}
    return {"config": name, "frames": F, "mode": plan["mode"], "core": plan["core"], "ms_per_batch": ms,
            "frames_per_s": F / ms * 1e3, "symbols_per_s": F * cfg.N / ms * 1e3,
            "phase_ms": [float(x) for x in phm], "pass1_tflops": p1, "pass2_tflops": p2,
            "pass1_frac": p1 / PEAK, "pass2_frac": p2 / PEAK, "frames_ok": float((st.cpu().numpy() == 0).mean()),
            "symbol_error_rate": ser, **extra}


def run_next(steps):
    """NEXT rows at C2 (65536 frames): soft boundaries + extrinsic overhead, and the Monte-Carlo loop."""
    from paper_1802_08483_b200 import phi
    cfg = bsidgen.configs()["C2"]
    F = BATCH["C2"]
    b = bsidgen.make_batch(cfg, 0, F)
    dev = torch.device("cuda", 0)
    d = Decoder.from_config(cfg, b.C, device=0)
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    a0 = phi(1, cfg.Pi, cfg.Pd, cfg.mt[0], cfg.mt[1], F, device=0)          # start-drift prior Phi_1
    bN = phi(cfg.tau, cfg.Pi, cfg.Pd, cfg.mt[0], cfg.mt[1], F, device=0)    # end drift Phi_tau
    d.decode(rx, off, rho, None, alpha0=a0, betaN=bN, extrinsic=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.decode(rx, off, rho, None, alpha0=a0, betaN=bN, extrinsic=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    out = [{"config": "C2+soft-boundaries+extrinsic (NEXT-1, NEXT-4)", "frames": F, "ms_per_batch": ms,
            "frames_per_s": F / ms * 1e3}]
    d.mc_run(cfg.seed, 0, 8192, 8192)
    ts = []
    for k in range(steps):
        t0 = time.perf_counter()
        res = d.mc_run(cfg.seed, 10_000_000 + k * F, F, 16384)
        ts.append(time.perf_counter() - t0)
    s = float(np.median(ts))
    out.append({"config": "C2 Monte-Carlo generate+decode+count (NEXT-3)", "frames": F, "ms_per_batch": s * 1e3,
                "frames_per_s": F / s, "symbol_error_rate": res["symbol_errors"] / (F * cfg.N),
                "frame_error_rate": res["frame_errors"] / F, "redraws": res["redraws"]})
    return out


def main():
    out = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "gpurun_out/sweep.json"
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 3
    res = []
    for name in ("C1", "C2", "C3", "C4", "C5"):
        for mode in ((0, 2, 1) if name in ("C1", "C2") else (0, 2)):
            t = time.time()
            try:
                r = run(name, mode, steps)
            except Exception as e:  # e.g. stored gamma does not fit
                r = {"config": name, "mode_arg": mode, "error": str(e)}
            r["wall_s"] = time.time() - t
            print(json.dumps(r), flush=True)
            res.append(r)
    for r in run_next(steps):
        print(json.dumps(r), flush=True)
        res.append(r)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
