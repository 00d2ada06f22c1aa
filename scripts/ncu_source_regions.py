"""Instruction and stall-sample shares per source line / line range from an ncu report:
python scripts/ncu_source_regions.py report.ncu-rep file.cu [N] [lo-hi:name ...]"""
import collections
import csv
import io
import subprocess
import sys

path, fsel = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
regions = []
for a in sys.argv[4:]:
    rng, name = a.split(":")
    lo, hi = rng.split("-")
    regions.append((int(lo), int(hi), name))
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
inst = collections.Counter()
samp = collections.Counter()
src = {}
fname = ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or not r[0]:
        continue
    key = (fname, int(r[0]))
    src[key] = r[1][:90]
    try:
        inst[key] += float(r[7] or 0)
        samp[key] += float(r[4] or 0)
    except (ValueError, IndexError):
        pass
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"total warp instructions {ti:.0f}, samples {ts:.0f}")
for lo, hi, name in regions:
    i = sum(v for (f, l), v in inst.items() if f == fsel and lo <= l < hi)
    s = sum(v for (f, l), v in samp.items() if f == fsel and lo <= l < hi)
    print(f"{name:24s} inst {100 * i / ti:5.1f}%  samples {100 * s / ts:5.1f}%")
for k, v in samp.most_common(n):
    print(f"{100 * v / ts:5.1f}% samples {100 * inst[k] / ti:5.1f}% inst  {k[0]}:{k[1]}  {src[k]}")
