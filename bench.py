#!/usr/bin/env python
"""Benchmark of the batched BSID MAP decoder (arXiv 1802.08483) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--mode auto|stored|recompute]
    python bench.py --impl reference ...      # the FP64 CPU oracle as the reference arm

One "step" = one decode_batch of the whole hot path (frame status -> lattice pass 1
-> alpha/beta -> lattice pass 2 (APP) -> normalisation) over the rank's frames.
Default workload: BASELINE.json configs[1] = C2 (q=16, n=10, N=100, Pi=Pd=0.01,
Ps=0.001), 65536 frames per GPU (weak scaling over ranks; frames are sharded with
no data-path collective).  Inputs are resident in HBM before timing; L2 is flushed
(256 MiB write) between timed steps, outside the per-step CUDA events.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import bsidgen  # noqa: E402

FP32_LANES_PER_SM = 128  # Blackwell SM: 4 SMSPs x 32 FP32 lanes


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=None, help="frames per GPU (default: the config's batch)")
    ap.add_argument("--total-frames", type=int, default=None,
                    help="strong scaling: this many frames for the whole job, split over the ranks")
    ap.add_argument("--mode", default="auto", choices=["auto", "stored", "recompute"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU work of the oracle sample")
    ap.add_argument("--N", type=int, default=None,
                    help="symbols per frame (default: the config's); keeps the config's code, channel and "
                         "drift limits -- a reduced-length test workload, not a bench line")
    ap.add_argument("--ws-limit-gb", type=float, default=None, help="cap the decoder workspace (chunking)")
    ap.add_argument("--dump", default=None, help="directory: each rank writes its L/status/frame range")
    return ap.parse_args()


def workload(args):
    import dataclasses
    cfg = bsidgen.all_configs()[args.config]
    if args.N is not None and args.N != cfg.N:
        cfg = dataclasses.replace(cfg, N=args.N, name=f"{cfg.name}@N{args.N}")
    return cfg


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi samples every 200 ms while the timed region runs."""
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=5)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# --------------------------------------------------------------------------- oracle leg

def oracle_frame_seconds(cfg):
    """Rough single-core oracle time of one full frame: 2 lattice passes x N x M_tau x q lattices x
    corridor cells, ~12 ns per FP64 cell; used only to size the sample."""
    cells = cfg.n * cfg.Mn - cfg.mn[0] * (cfg.mn[0] - 1) // 2
    return 2 * cfg.N * cfg.Mt * cfg.q * cells * 12e-9


class OracleSampler:
    """Times the FP64 oracle, as it stands, on the host cores over whole frames of the workload.
    Short frames: one frame per host thread (frames in parallel).  Long frames (single-core estimate
    above the target, C4/C5): one frame at a time with the oracle's in-frame threads on every core
    (its m' loops; bit-identical to the serial oracle) -- at least one FULL frame is always timed,
    so C5's baseline is a full N = 10^4 frame (minutes), never an extrapolation."""

    def __init__(self, cfg, target_seconds):
        import oracle
        self.cfg = cfg
        self.threads = os.cpu_count() or 1
        self.prob = oracle.Problem(cfg.q, cfg.n, cfg.N, bsidgen.codebook(cfg), cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
        est = oracle_frame_seconds(cfg)
        self.in_frame = est > target_seconds
        if self.in_frame:
            self.count = 1
            self.how = f"one frame at a time, {self.threads} oracle threads inside the frame"
            dt = self.run(10_000_000, 1)
            self.count = int(max(1, min(64, target_seconds / dt)))
        else:
            probe = self.threads
            dt = self.run(10_000_000, probe)
            self.count = max(self.threads, int(target_seconds / max(dt / probe, 1e-9)) // self.threads * self.threads)
            self.count = min(self.count, 4096)
            self.how = f"{self.threads} host threads over frames"
        self.probe_s = dt

    def run(self, first, count):
        import oracle
        b = bsidgen.make_batch(self.cfg, first, count, C=self.prob.C)
        ys = [b.bits(f) for f in range(count)]
        pl = [b.priors[f].astype(np.float64) if b.priors is not None else None for f in range(count)]
        t0 = time.perf_counter()
        if self.in_frame:
            oracle.set_threads(self.threads)
            try:
                for y, pr in zip(ys, pl):
                    oracle.decode(self.prob, y, pr)
            finally:
                oracle.set_threads(1)
        else:
            oracle.decode_many(self.prob, ys, pl, self.threads)
        return time.perf_counter() - t0


def cpu_baseline(cfg, target_seconds):
    o = OracleSampler(cfg, target_seconds)
    if o.in_frame and o.count == 1:
        dt, count = o.probe_s, 1   # the probe already timed one full frame
    else:
        count = o.count
        dt = o.run(20_000_000, count)
    return {"value": count / dt, "unit": "frames/s", "cores": o.threads, "kind": "oracle",
            "sample": f"{count} full frames of {cfg.name} (global frame indices 10000000.. / 20000000..), "
                      f"FP64 C oracle, {o.how}, {dt:.1f} s"}


def reference_arm(args, cfg):
    from paper_1802_08483_b200.sharding import dist_env
    rank, world, _ = dist_env()
    if rank != 0:
        return
    per_step = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    o = OracleSampler(cfg, per_step)
    count = o.count
    for w in range(args.warmup):
        o.run(30_000_000 + w * count, count)
    times = [o.run(40_000_000 + s * count, count) for s in range(args.steps)]
    total = sum(times)
    value = count * args.steps / total  # frames/s of the configuration, whole frames timed
    line = {
        "impl": "reference", "metric": "frames/s", "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": describe(cfg), "frames_per_step": count, "sample": "bounded oracle sample of full frames"},
        "symbols_per_s": value * cfg.N,
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": o.threads, "kind": "oracle",
                         "sample": f"{count} full frames x {args.steps} steps of {cfg.name}, FP64 C oracle, {o.how}"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def describe(cfg):
    return (f"{cfg.name}: q={cfg.q} n={cfg.n} N={cfg.N} Pi={cfg.Pi} Pd={cfg.Pd} Ps={cfg.Ps} "
            f"m_n=[{cfg.mn[0]},{cfg.mn[1]}] m_tau=[{cfg.mt[0]},{cfg.mt[1]}] "
            f"priors={'non-uniform' if cfg.priors else 'uniform'}")


# ------------------------------------------------------------------------- roofline inputs

def fp32_peak(sms):
    """FP32 peak of the ALU roofline: the measured FFMA2 throughput of this B200 pool
    (profiles/fp32_peak.json, tools/ubench/fp32_peak.cu: independent FFMA2 chains on every SM);
    MEASURED_PEAKS.json has no FP32 entry.  Fallback: the guide's unit counts at the max SM clock."""
    path = os.path.join(ROOT, "profiles", "fp32_peak.json")
    nominal = sms * FP32_LANES_PER_SM * 2 * 1965e6 / 1e12
    try:
        m = json.load(open(path))
        return float(m["ffma2_tflops"]), (f"measured: FFMA2 microbenchmark {m['ffma2_tflops']:.1f} TFLOP/s at "
                                          f"{m.get('sm_mhz_nvidia_smi_under_load', '?')} MHz (profiles/fp32_peak.json; nominal "
                                          f"{nominal:.1f} = {sms} SMs x 128 lanes x 2 flop x 1965 MHz)")
    except (OSError, KeyError, ValueError):
        return nominal, (f"nominal: {sms} SMs x 128 FP32 lanes x 2 flop x 1965 MHz (no profiles/fp32_peak.json; "
                         "MEASURED_PEAKS.json has no FP32 entry)")


def ncu_profile(cfg, key, frames, plan):
    """DRAM traffic and executed FP32 flops of the dominant kernel from one `ncu --set full` capture
    (profiles/ncu_summary.json, tools/ncu_summary.py) -- used only if it was captured at this source
    digest, for this workload and batch (else null, with the reason)."""
    from paper_1802_08483_b200._lib import source_digest
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    digest = source_digest()
    try:
        ent = json.load(open(path)).get(cfg.name, {}).get(key)
    except (OSError, ValueError):
        ent = None
    if not ent:
        return {"traffic": None, "ncu": f"no capture of {cfg.name}/{key} in profiles/ncu_summary.json"}
    if ent.get("src_digest") != digest or ent.get("frames") != frames:
        return {"traffic": None, "ncu": f"stale: capture {ent.get('round')} at source digest {ent.get('src_digest')}, "
                                        f"{ent.get('frames')} frames; this run {digest}, {frames} frames"}
    out = {"traffic": ent.get("dram_bytes_per_launch"), "ncu": f"{ent.get('round')} (source digest {digest})",
           "fma_pipe_active_ncu": ent.get("fma_pipe_active")}
    if ent.get("fp32_flops_executed"):
        out["executed_flops_per_launch"] = ent["fp32_flops_executed"]
    return out


# ------------------------------------------------------------------------------ our arm

def main():
    args = parse()
    cfg = workload(args)
    if args.impl == "reference":
        return reference_arm(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_1802_08483_b200 import Decoder, MODE_AUTO, MODE_RECOMPUTE, MODE_STORED
    from paper_1802_08483_b200.sharding import (barrier, dist_env, frame_range, frame_range_strong, max_over_ranks,
                                                sum_over_ranks)

    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # one process per GPU (LOCAL_RANK); BSIDMAP_DIST_BACKEND=gloo and the modulo over the visible
    # devices let the multi-rank path run with several ranks on one GPU (a functional check only)
    backend = os.environ.get("BSIDMAP_DIST_BACKEND", "nccl")
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    local = dev.index
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    frames = args.frames or cfg.frames
    strong = args.total_frames is not None
    first, count = frame_range_strong(rank, world, args.total_frames) if strong else frame_range(rank, world, frames)
    b = bsidgen.make_batch(cfg, first, count)
    mode = {"auto": MODE_AUTO, "stored": MODE_STORED, "recompute": MODE_RECOMPUTE}[args.mode]
    d = Decoder.from_config(cfg, b.C, mode=mode, device=local)
    if args.ws_limit_gb:
        d.set_workspace_limit(int(args.ws_limit_gb * 2**30))
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    L = torch.empty((count, cfg.N, cfg.q), dtype=torch.float32, device=dev)
    st = torch.empty((count,), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    plan = d.plan(count)

    d.set_timing(True)
    for _ in range(args.warmup):
        d.decode_batch(rx, off, rho, pri, L, st, stream)
    torch.cuda.synchronize(dev)

    nodes = d.lattice_nodes()
    # windows with 0 <= n i + m' <= rho, per lattice pass, of the frames the phase events time: the
    # library's phase events bracket the FIRST chunk's kernels when the batch is chunked
    lattices = d.valid_lattices(b.rho[:plan["chunk"]])
    flops_per_lattice = 5 * nodes - cfg.Mn       # P:857 node count; 3 mul + 2 add per node, last row 3 flops
    flops_pass = lattices * flops_per_lattice

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phases, launches = [], 0
    clocks = ClockSampler(local)
    barrier(dev)
    torch.cuda.synchronize(dev)
    clocks.start()
    for s in range(args.steps):
        flush.zero_()
        ev[s][0].record(stream)
        d.decode_batch(rx, off, rho, pri, L, st, stream)
        ev[s][1].record(stream)
        phases.append(d.phase_times())   # synchronises the stream (per-step device timing only)
        launches += d.last_launch_count()
    torch.cuda.synchronize(dev)
    barrier(dev)
    clk = clocks.stop()
    step_ms = [a.elapsed_time(bb) for a, bb in ev]
    local_ms = sum(step_ms)
    max_ms = max_over_ranks(local_ms, dev)
    total_frames = sum_over_ranks(count * args.steps, dev)
    value = total_frames / (max_ms / 1e3)

    # roofline of the dominant kernel: lattice pass 1 vs pass 2, whichever takes longer on average
    ph = np.array(phases)  # [steps][6]: init, pass 1, exposed alpha/beta, pass 2, finalize, alpha/beta busy
    mean_ph = ph.mean(0)
    dominant = 1 if mean_ph[1] >= mean_ph[3] else 3
    slab = plan["mode"] == "recompute-slab"
    if slab:  # phases: [1] forward sweep (every pass-1 slab, alpha overlapped), [3] backward sweep
        dominant = 1
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_tf, peak_basis = fp32_peak(sms)
    achieved = flops_pass / (mean_ph[dominant] / 1e3) / 1e12
    prof = ({"ncu": "not captured for the slab schedule (the ncu entries are the Gamma-sum kernels)"} if slab else
            ncu_profile(cfg, "lattice_pass1" if dominant == 1 else "lattice_pass2", count, plan))
    if "executed_flops_per_launch" in prof:  # executed work over the same live launch time
        prof["executed_achieved"] = prof["executed_flops_per_launch"] / (mean_ph[dominant] / 1e3) / 1e12
        prof["frac_executed"] = prof["executed_achieved"] / peak_tf

    # end-to-end through the host-buffer C-ABI entry (pinned buffers, copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        h_rx = torch.from_numpy(b.rx.ravel().copy()).pin_memory()
        h_off = torch.from_numpy(b.offsets).pin_memory()
        h_rho = torch.from_numpy(b.rho).pin_memory()
        h_pri = torch.from_numpy(b.priors).pin_memory() if b.priors is not None else None
        h_L = torch.empty((count, cfg.N, cfg.q), dtype=torch.float32).pin_memory()
        h_st = torch.empty((count,), dtype=torch.int32).pin_memory()
        d.set_timing(False)
        d.decode_host(h_rx, h_off, h_rho, h_pri, h_L, h_st, stream)  # warm the staging buffers
        barrier(dev)
        torch.cuda.synchronize(dev)
        t_e2e = []
        for s in range(max(1, min(args.steps, 5))):
            flush.zero_()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            d.decode_host(h_rx, h_off, h_rho, h_pri, h_L, h_st, stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            t_e2e.append(e0.elapsed_time(e1))
        e_ms = max_over_ranks(sum(t_e2e), dev)
        e_frames = sum_over_ranks(count * len(t_e2e), dev)
        h2d = h_rx.numel() * 4 + h_off.numel() * 8 + h_rho.numel() * 4 + (h_pri.numel() * 4 if h_pri is not None else 0)
        d2h = h_L.numel() * 4 + h_st.numel() * 4
        e2e = {"value": e_frames / (e_ms / 1e3), "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}
        ok = (h_st.numpy() == 0).mean()
        if ok < 0.999 and rank == 0:
            print(f"warning: only {ok:.4f} of frames decoded OK in e2e", file=sys.stderr)

    plan_after = d.plan(count)
    st_h = st.cpu().numpy()
    L_h = L.cpu().numpy()
    if args.dump:
        os.makedirs(args.dump, exist_ok=True)
        np.savez(os.path.join(args.dump, f"rank{rank}.npz"), L=L_h, status=st_h, first=first, count=count)
    # job-wide symbol errors and decoded frames: summed over ranks (each rank holds its own shard)
    sym_err = sum_over_ranks(int((np.argmax(L_h, 2) != b.msg).sum()), dev)
    frames_ok = sum_over_ranks(int((st_h == 0).sum()), dev)
    job_frames = sum_over_ranks(count, dev)
    ser = sym_err / max(1.0, job_frames * cfg.N)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(cfg, args.cpu_seconds)
        line = {
            "metric": "frames/s", "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32",
"dtype_detail": "FP32: lattice / gamma / Gamma (receiver metric, P:272-275) and each window's APP term "
                            "alpha*beta*gamma; FP64: alpha/beta recursions and normalisation, the APP sum over "
                            "windows and symbols, and the L normalisation (output FP32)",
            "data": "synthetic",
            "config": {"workload": describe(cfg), "frames_per_gpu": count,
                       "total_frames": int(total_frames // args.steps), "mode": plan["mode"],
                       "core": plan["core"], "chunks": plan["chunks"], "parallelism": f"frames sharded x{world}",
                       "app_frames_per_warp": plan_after.get("app_frames_per_warp"),
                       "l2": "flushed (256 MiB write) between timed steps; per-step working set > L2"},
            "symbols_per_s": value * cfg.N,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": prof.get("traffic"),
                         "kernel": ("slab forward sweep (pass 1 of every slab, alpha overlapped)" if slab else
                                    "lattice pass 1 (k_gamma_sum)" if dominant == 1 else "lattice pass 2 (k_app)"),
                         "peak_basis": peak_basis,
                         "flops_per_launch": flops_pass, "launch_ms": float(mean_ph[dominant]),
                         "frames_per_launch": int(min(plan["chunk"], count)),
                         "note": "achieved/frac count the paper's algorithmic work, 5 flops per lattice node over "
                                 "the P:857 node count of every valid lattice (algorithmic-equivalent); the kernel "
                                 "executes fewer (2 FFMA per node after the exact G = F/Pd^r rescaling, suffix "
                                 "classes, prefix sharing, folded rows, skipped all-zero tiles): executed_* are the "
                                 "FP32 flops ncu counted for this kernel at this source digest over the same "
                                 "live launch time",
                         **{k: v for k, v in prof.items() if k != "traffic"}},
            "phase_ms": {"init": float(mean_ph[0]), "lattice_pass1": float(mean_ph[1]),
                         "alpha_beta": float(mean_ph[2]), "lattice_pass2": float(mean_ph[3]),
                         "finalize": float(mean_ph[4]),
                         "alpha_beta_busy": float(mean_ph[5]) if len(mean_ph) > 5 else float(mean_ph[2]),
                         **({"note": "slab schedule: lattice_pass1 = forward sweep (pass 1 + alpha per slab), "
                                     "lattice_pass2 = backward sweep (pass 1 where alpha != 0, beta, live APP)"}
                            if slab else {})},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "frames_ok": frames_ok / max(1.0, job_frames),
            "symbol_error_rate": ser,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
