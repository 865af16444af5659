"""Aggregate an ncu --set full report's warp-stall samples per CUDA source line (needs -lineinfo).
Usage: python tools/ncu_src_lines.py report.ncu-rep [top_n] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep] + kf + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
recs, tot, cur = [], 0, None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iS = r.index("Warp Stall Sampling (All Samples)")
        iN = r.index("Warp Stall Sampling (Not-issued Samples)")
        iI = r.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    # a source line with commas / quotes may split into extra fields: index the metrics from the end
    extra = len(r) - len(hdr)
    def col(i):
        return r[i + extra] if extra > 0 else r[i]
    try:
        v = int(col(iS))
    except ValueError:
        continue
    ni = col(iN)
    ins = col(iI)
    tot += v
    recs.append((v, int(ni) if ni.isdigit() else 0, int(ins) if ins.isdigit() else 0, cur, r[0],
                 ",".join(r[1:2 + max(extra, 0)]).strip()[:100]))
recs.sort(reverse=True)
print("total samples %d" % tot)
print("%7s %6s %7s %12s  %s" % ("samples", "%", "notiss", "warp-instr", "file:line source"))
for v, ni, ins, f, l, s in recs[:top]:
    print("%7d %5.1f%% %7d %12d  %s:%s %s" % (v, 100.0 * v / max(tot, 1), ni, ins, f, l, s))
