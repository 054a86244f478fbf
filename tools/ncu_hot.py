"""Print the hottest SASS lines (warp-stall samples) of a kernel from an ncu report.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in data)
print("total samples", tot, "sass lines", len(data))
for k, r in enumerate(data):
    r.append(k)
for r in sorted(data, key=lambda r: -int(r[si] or 0))[:top]:
    print(f"{int(r[si]):7d} {100*int(r[si])/max(tot,1):5.1f}%  #{r[-1]:5d} exec={r[ie]:>10s}  {r[1][:90]}")
