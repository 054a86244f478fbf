"""Summarise an ncu --set full report and a launch list into profiles/.
usage: python tools/ncu_summary.py <tag> <gpurun_out/dir> <config> <frames> [--no-write]
--no-write: print the summary only (on the GPU box); the report is read from prof.ncu-rep or, when
that was deleted, from raw.csv (ncu --page raw --csv) in the same directory.
The capture directory holds digest.txt (the library source digest at capture time, tools/gpu_prof.sh);
bench.py uses an entry only at the same digest and batch size."""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

tag, src, cfg, frames = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
digest = open(os.path.join(src, "digest.txt")).read().strip()
FP32_OPS = {"ffma": 2, "ffma2": 4, "fadd": 1, "fadd2": 2, "fmul": 1, "fmul2": 2}
FP64_OPS = {"dfma": 2, "dadd": 1, "dmul": 1}
os.makedirs("profiles", exist_ok=True)
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size"] + \
          [f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum" for o in list(FP32_OPS) + list(FP64_OPS)]
NO_WRITE = "--no-write" in sys.argv
if os.path.exists(os.path.join(src, "prof.ncu-rep")):
    raw = subprocess.run(["ncu", "-i", os.path.join(src, "prof.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
else:
    raw = open(os.path.join(src, "raw.csv")).read()
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
kernels = []
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            d[m] = (r[hdr.index(m)], units[hdr.index(m)])
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): r[hdr.index(h)] for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")}
    top = sorted(((float(v or 0), k) for k, v in stalls.items() if v not in ("", "n/a")), reverse=True)[:6]
    d["top_stalls"] = [(k, int(v)) for v, k in top]
    kernels.append(d)

def gb(v):
    val, unit = v
    try:
        x = float(val)
    except ValueError:
        return None
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)

summ = json.load(open("profiles/ncu_summary.json")) if os.path.exists("profiles/ncu_summary.json") else {}
entry = summ.setdefault(cfg, {})
lines = [f"# ncu summary {tag} ({cfg}, bench launch configuration)", "",
         f"Source: `ncu --set full --clock-control none` of `python bench.py --config {cfg} --steps 1 --warmup 0`.",
         "Per-launch device times under ncu are cold-cache and serialised: compare shares, not absolutes.", ""]
for d in kernels:
    name = d["kernel"]
    key = ("lattice_pass1" if "gamma_sum" in name else "lattice_pass2" if "k_app" in name else
           "live" if "k_live" in name else "alpha_beta")
    rd, wr = gb(d.get("dram__bytes_read.sum", ("", ""))), gb(d.get("dram__bytes_write.sum", ("", "")))
    fp = d.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", ("", ""))[0]
    try:
        fp = float(fp) / 100.0
    except ValueError:
        fp = None
    def ops(table):
        tot = 0.0
        for o, w in table.items():
            v = d.get(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum", ("", ""))[0].replace(",", "")
            try:
                tot += w * float(v)
            except ValueError:
                return None
        return tot
    entry[key] = {"kernel": name, "dram_bytes_per_launch": (rd + wr) if rd is not None and wr is not None else None,
                  "time_ms": float(d["gpu__time_duration.sum"][0].replace(",", "")) if "gpu__time_duration.sum" in d else None,
                  "fma_pipe_active": fp, "fp32_flops_executed": ops(FP32_OPS), "fp64_flops_executed": ops(FP64_OPS),
                  "round": tag, "src_digest": digest, "frames": frames}
    lines.append(f"## {name}")
    for m in METRICS:
        if m in d:
            lines.append(f"- {m}: {d[m][0]} {d[m][1]}")
    lines.append(f"- top stall reasons (pc samples): {d['top_stalls']}")
    lines.append("")
launch_csv = os.path.join(src, "launches.csv")
if os.path.exists(launch_csv):
    body = [l for l in open(launch_csv) if l.startswith('"')]
    rr = list(csv.reader(io.StringIO("".join(body))))
    h = rr[0]
    t = defaultdict(list)
    for r in rr[1:]:
        t[r[h.index("Kernel Name")]].append(float(r[h.index("Metric Value")].replace(",", "")))
    tot = sum(sum(v) for k, v in t.items() if "bsidmap" in k)
    lines += ["## launch list (gpu__time_duration.sum, ns)", "", "| kernel | launches | mean ms | share of decode |", "|---|---|---|---|"]
    for k, v in t.items():
        share = f"{100 * sum(v) / tot:.1f}%" if "bsidmap" in k else "-"
        lines.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v) / 1e6:.3f} | {share} |")
    if not NO_WRITE:
        open(f"profiles/{tag}_{cfg}_launches.csv", "w").write("".join(body))
if not NO_WRITE:
    open(f"profiles/{tag}_ncu_{cfg}.md", "w").write("\n".join(lines) + "\n")
    json.dump(summ, open("profiles/ncu_summary.json", "w"), indent=1)
print("\n".join(lines))
