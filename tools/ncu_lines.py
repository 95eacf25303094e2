"""Per-source-line warp-stall sample share from an ncu report (--import-source on).

usage: python tools/ncu_lines.py report.ncu-rep [top]
"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, last, tot = None, None, 0.0
agg, src = collections.Counter(), {}
for r in csv.reader(io.StringIO(txt)):
    if not r or r[0] in ("Function Name", "Line No"):
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    try:
        s = float(r[4]) if len(r) > 4 and r[4] else 0.0
    except ValueError:
        s = 0.0
    if r[0]:
        last = (cur, int(r[0]))
        src[last] = r[1].strip()[:90]
    if last is not None:
        agg[last] += s
        tot += s
print("total samples", tot)
for k, v in agg.most_common(top):
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]} {src.get(k, '')}")
