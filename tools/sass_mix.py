"""Dynamic SASS instruction mix of one kernel from an ncu report (source page, SASS view):
share of executed warp instructions and of warp-stall samples per opcode.
usage: python tools/sass_mix.py <report.ncu-rep> <kernel regex> [top]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
cnt, stall = collections.Counter(), collections.Counter()
hdr = None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    src = r[hdr.index("Source")].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    op = op.split(".")[0]
    try:
        cnt[op] += int(r[hdr.index("Instructions Executed")] or 0)
        stall[op] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        pass
tot, stot = sum(cnt.values()) or 1, sum(stall.values()) or 1
print(f"executed warp instructions: {tot}")
for op, n in cnt.most_common(top):
    print(f"{op:10s} {100 * n / tot:6.2f}% of executed   {100 * stall[op] / stot:6.2f}% of stall samples")
