"""DRAM traffic per launch of the bench components from `ncu --set full` reports:
python scripts/traffic_from_ncu.py PROFDIR OUT.json

PROFDIR holds full_c<config>_<name>.csv (the raw page, exported by scripts/profile_round.sh) or
.ncu-rep.  Each bench component
(Solver::profile names) maps to the kernels one launch of it runs; its traffic is the sum of
their dram__bytes_read.sum + dram__bytes_write.sum.  bench.py reads OUT.json (profiles/
r*_traffic*.json) and reports a component's traffic only when every listed kernel is in the
plan's captured solve graph."""
import csv
import io
import json
import os
import subprocess
import sys

COMPONENTS = {  # (config, component): [report names]
    (1, "update_residual"): ["update"], (1, "hole2d_fused_dmma"): ["hole"], (1, "slabstep2d"): ["slabstep"],
    (1, "step_dots_skeleton"): ["dots"],
    (2, "update_residual"): ["update"], (2, "hole_backtransform_dmma"): ["back"], (2, "slab2d_fwd_pcr"): ["slabfwd"],
    (2, "hole2d_mode_lines_separators_strip_lines"): ["lines"],
    (3, "update_residual"): ["axpy", "cand"], (3, "hole_fill"): ["hole"], (3, "residual"): ["cand"],
    (4, "update_residual"): ["axpy", "cand"], (4, "hole_fill"): ["hole"], (4, "residual"): ["cand"],
}


def kernel_name(raw):
    """`stencil2d_ym_kernel<1,0>` from ncu's `void unnamed>::stencil2d_ym_kernel<1, 0>(MarchArgs, int)`
    (bench.py normalizes the library's own demangled names the same way)."""
    n = raw.replace("(anonymous namespace)::", "")
    if "unnamed>::" in n:
        n = n.split("unnamed>::", 1)[1]
    if n.startswith("void "):
        n = n[5:]
    depth = 0
    for i, ch in enumerate(n):
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            n = n[:i]
            break
    return n.replace(" ", "").replace("false", "0").replace("true", "1")


def read(path):
    if path.endswith(".csv"):  # the raw page already exported on the GPU box (profile_round.sh)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, r = rows[0], rows[1], rows[2]

    def val(m):
        i = hdr.index(m)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
        return float(r[i].replace(",", "")) * scale
    return {"kernel": kernel_name(r[hdr.index("Kernel Name")]), "dram_read_bytes": val("dram__bytes_read.sum"),
            "dram_write_bytes": val("dram__bytes_write.sum")}


def main(d, out_path):
    res = {"source": os.path.basename(os.path.normpath(d)), "kernels": {}}
    for (cid, comp), names in COMPONENTS.items():
        parts = []
        for n in names:
            p = os.path.join(d, f"full_c{cid}_{n}.csv")
            if not os.path.exists(p):
                p = os.path.join(d, f"full_c{cid}_{n}.ncu-rep")
            if not os.path.exists(p):
                break
            parts.append(read(p))
        else:
            res["kernels"][f"{cid}/{comp}"] = {
                "kernels": [x["kernel"] for x in parts],
                "dram_read_bytes": sum(x["dram_read_bytes"] for x in parts),
                "dram_write_bytes": sum(x["dram_write_bytes"] for x in parts)}
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
