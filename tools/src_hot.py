"""Per-CUDA-source-line share of executed warp instructions and warp-stall samples of one kernel
(ncu --page source --print-source cuda,sass, from a kept report).
usage: python tools/src_hot.py <report.ncu-rep> <kernel regex> [top]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
fname, hdr, line, text = None, None, None, {}
smp, ins = collections.Counter(), collections.Counter()
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a CUDA source line (its SASS rows follow with an empty line number)
        line = (fname, int(r[0]))
        text[line] = r[1].strip()
    if line is None or not r[2].startswith("0x"):
        continue
    try:
        smp[line] += int(r[4] or 0)
        ins[line] += int(r[7] or 0)
    except ValueError:
        pass
ts, ti = sum(smp.values()) or 1, sum(ins.values()) or 1
print(f"stall samples {ts}, executed warp instructions {ti}")
for ln, s in smp.most_common(top):
    print(f"{100 * s / ts:5.1f}% smp {100 * ins[ln] / ti:5.1f}% ins  {ln[0]}:{ln[1]:<4} {text.get(ln, '')[:90]}")
