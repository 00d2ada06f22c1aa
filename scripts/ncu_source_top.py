"""Top source lines by warp-stall samples from an ncu report (--page source, cuda+sass):
python scripts/ncu_source_top.py report.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.Counter()
srcline = {}
fname = ""
total = 0
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:  # a source line row
        cur = (fname, r[0])
        srcline[cur] = r[1][:100]
        try:
            v = float(r[4] or 0)
        except (ValueError, IndexError):
            v = 0
        agg[cur] += v
        total += v
for (f, ln), v in agg.most_common(n):
    print(f"{100 * v / max(total, 1):5.1f}%  {f}:{ln}  {srcline[(f, ln)]}")
