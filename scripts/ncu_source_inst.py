"""Top source lines by executed warp instructions (and stall samples) from an ncu report:
python scripts/ncu_source_inst.py report.ncu-rep [N]"""
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
hdr = None
inst = collections.Counter()
samp = collections.Counter()
src = {}
fname = ""
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    src[key] = r[1][:90]
    try:
        inst[key] += float(r[7] or 0)
        samp[key] += float(r[4] or 0)
    except (ValueError, IndexError):
        pass
ti = sum(inst.values()) or 1
ts = sum(samp.values()) or 1
print(f"total warp instructions {ti:.3e}")
for k, v in inst.most_common(n):
    print(f"{100 * v / ti:5.1f}% inst {100 * samp[k] / ts:5.1f}% stall  {k[0]}:{k[1]}  {src[k]}")
