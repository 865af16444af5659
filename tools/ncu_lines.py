"""Summarise an ncu report by CUDA source line: share of warp-stall samples, top stall
reasons, instructions executed.  Usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
fname = None
agg = {}
for x in rows:
    if x and x[0] == "File Path":
        fname = x[1].split("/")[-1]
        continue
    if x and x[0] == "Line No":
        hdr = x
        continue
    if not hdr or len(x) < 6 or x[2] != "-":
        continue
    d = {c[6:]: int(x[i]) for i, c in enumerate(hdr)
         if c.startswith("stall_") and "Not Issued" not in c and x[i].isdigit()}
    ie = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
    agg[(fname, int(x[0]), x[1].strip()[:64])] = (d, int(x[ie] or 0) if ie is not None else 0)
tot = sum(sum(d.values()) for d, _ in agg.values()) or 1
toti = sum(i for _, i in agg.values()) or 1
print("samples %d  instructions %d" % (tot, toti))
for k, (d, ins) in sorted(agg.items(), key=lambda kv: -sum(kv[1][0].values()))[:N]:
    s = sum(d.values())
    top = ", ".join("%s %d" % kv for kv in sorted(d.items(), key=lambda kv: -kv[1])[:3])
    print("%5.1f%% %5.1f%%i %s:%d %-64s %s" % (100 * s / tot, 100 * ins / toti, k[0], k[1], k[2], top))
