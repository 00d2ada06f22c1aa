"""Copy one profiling pass (scripts/profile_round.sh TAG bench|full, merged back under
gpurun_out/prof_TAG) into profiles/ under a round/version name:

    python scripts/collect_profiles.py TAG r2 v5

writes profiles/<round>_bench_<ver>.json, <round>_bench_ref_<ver>.json, the launch lists
<round>_launches_c{1..4}_<ver>.csv with their summaries, the raw ncu metric pages transposed to
(metric, unit, value) rows under <round>_ncu_raw_<ver>/, the DRAM traffic per bench component
<round>_traffic_<ver>.json (what bench.py's roofline.traffic reads) and the per-config kernel
tables /tmp/ncu_tables_<ver>.md for the summary file's body."""
import csv
import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(tag, rnd, ver):
    src = os.path.join(ROOT, "gpurun_out", f"prof_{tag}")
    prof = os.path.join(ROOT, "profiles")
    for a, b in (("bench.json", f"{rnd}_bench_{ver}.json"), ("bench_ref.json", f"{rnd}_bench_ref_{ver}.json")):
        if os.path.exists(os.path.join(src, a)):
            shutil.copy(os.path.join(src, a), os.path.join(prof, b))
    for c in (1, 2, 3, 4):
        p = os.path.join(src, f"launches_c{c}.csv")
        if not os.path.exists(p):
            continue
        dst = os.path.join(prof, f"{rnd}_launches_c{c}_{ver}.csv")
        shutil.copy(p, dst)
        rel = os.path.relpath(dst, ROOT)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_summary.py"), rel],
                             capture_output=True, text=True, cwd=ROOT).stdout
        open(dst.replace(".csv", "_summary.txt"), "w").write(out)
    raw = os.path.join(prof, f"{rnd}_ncu_raw_{ver}")
    pages = sorted(glob.glob(os.path.join(src, "full_c*.csv")))
    if pages:
        os.makedirs(raw, exist_ok=True)
    for p in pages:
        rows = list(csv.reader(open(p)))
        if len(rows) < 3:
            print("empty page", p)
            continue
        with open(os.path.join(raw, os.path.basename(p).replace("full_", "")), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["metric", "unit", "value"])
            for h, u, v in zip(rows[0], rows[1], rows[2]):
                w.writerow([h, u, v])
    if pages:
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "traffic_from_ncu.py"), src,
                        os.path.join(prof, f"{rnd}_traffic_{ver}.json")], capture_output=True, cwd=ROOT)
        with open(f"/tmp/ncu_tables_{ver}.md", "w") as f:
            for c in (1, 2, 3, 4):
                f.write(f"## Config {c}\n")
                first = True
                for p in sorted(glob.glob(os.path.join(src, f"full_c{c}_*.csv"))):
                    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), p],
                                         capture_output=True, text=True).stdout.strip().split("\n")
                    f.write("\n".join(out[-3:] if first else out[-1:]) + "\n")
                    first = False
        print("tables:", f"/tmp/ncu_tables_{ver}.md")


if __name__ == "__main__":
    main(*sys.argv[1:4])
