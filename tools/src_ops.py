"""Executed warp instructions of one kernel by (CUDA source line, SASS opcode), from a kept ncu report
(--page source --print-source cuda,sass): where the MOVs, branches and loads come from.
usage: python tools/src_ops.py <report.ncu-rep> <kernel regex> [opcode ...]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
want = set(sys.argv[3:]) or {"MOV", "BRA", "LDS", "UMOV", "R2UR", "ISETP", "UISETP"}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
fname, hdr, line, text = None, None, None, {}
cnt = collections.Counter()
tot = 0
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
    if r[0]:
        line = (fname, int(r[0]))
        text[line] = r[1].strip()
    if line is None or not r[2].startswith("0x"):
        continue
    op = r[3].strip().split()[0] if r[3].strip() else "?"
    if op.startswith("@"):
        op = r[3].strip().split()[1]
    op = op.split(".")[0]
    try:
        n = int(r[7] or 0)
    except ValueError:
        continue
    tot += n
    cnt[(line, op)] += n
print(f"executed warp instructions: {tot}")
byop = collections.Counter()
for (l, op), n in cnt.items():
    byop[op] += n
for op, n in byop.most_common(20):
    print(f"{op:8s} {100 * n / max(1, tot):6.2f}%")
for op in sorted(want):
    rows = sorted(((n, l) for (l, o), n in cnt.items() if o == op), reverse=True)[:12]
    if not rows:
        continue
    print(f"\n== {op}: top source lines")
    for n, l in rows:
        print(f"{100 * n / max(1, tot):6.2f}%  {l[0]}:{l[1]}  {text.get(l, '')[:90]}")
