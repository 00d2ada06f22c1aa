"""ASDSM benchmark on B200.

Metric: fine-grid DOF-iterations/s = (fine unknowns x ASDSM iterations) / solve time.  One
"step" = one full ASDSM solve of a BASELINE.json problem (initial guess + K iterations, K from
BASELINE.json), on a prebuilt plan (the reference's SolverContext: tables, operators) with the
assembled right-hand-side bundle resident in HBM; L2 flushed between steps.  `e2e`: the same
solve through the C-ABI (asdsm_solve) with pinned HOST buffers (H2D of the bundle, D2H of u, r
and the history inside the timed region).

The headline line is `--config` (default 1, BASELINE configs[1]); with the default
`--per-config`, every BASELINE config is measured the same way (value, e2e, rooflines, clocks,
a bounded CPU sample of the reference) and listed under "per_config".

  python bench.py [--config 1] [--steps K] [--warmup W] [--gpus N] [--impl ours|reference]

The reference arm (--impl reference) runs the reference's own C++ sources (oracle/_ref) on the
host cores; it does not import this package.
"""
import argparse
import ctypes
import glob
import json
import os
import re
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))

# Workload names carry the mesh actually run: the reference needs (N_f + 1) = n (N_c + 1)
# (mesh.cpp:63-68), so each BASELINE N maps to the nearest admissible N_f at the reference's
# default N_c = 9.
CONFIG_NAMES = [
    "2d_steady_Nf129_Nc9_manufactured",
    "2d_steady_Nf1029_Nc9_bumps8",
    "2d_advection_Nf4099_Nc9_bumps16",
    "3d_steady_Nf259_Nc9_manufactured",
    "2d_time_Nf509_Nc9_spacetime_bumps8",
]
ITERATIONS = [10, 20, 20, 10, 10]
# fine / coarse interior counts per axis of each config (include/asdsm_problems.hpp baseline_mesh)
MESHES = [([129, 129], [9, 9]), ([1029, 1029], [9, 9]), ([4099, 4099], [9, 9]), ([259] * 3, [9] * 3),
          ([509] * 3, [9] * 3)]


def config_dict(cid, world):
    """The `config` object of both arms (identical keys and values)."""
    fine, coarse = MESHES[cid]
    return {"workload": CONFIG_NAMES[cid], "config_id": cid, "fine_counts": fine, "coarse_counts": coarse,
            "iterations": ITERATIONS[cid], "dof": int(np.prod(fine)),
            "l2": "GPU arm: flushed between steps (256 MB write)",
            "parallelism": f"replicas x{world}" if world > 1 else "1gpu"}
# Bounded CPU samples of the reference per config: (nf, nc, iterations run, what).  Full solves
# where they take seconds; the full mesh with 1 iteration for config 2 (the rate of a K-iteration
# solve is extrapolated from the measured initial-guess and iteration times).  The 3D meshes do
# not fit a bounded sample on the host (the reference factors three 9 x 259 x 259 slabs and a
# 25^3 / 50^3 hole block with a band LU: hours), so config 3 is sampled on 103^3 at N_c = 3 (the
# config's 25^3 holes) and config 4 on 81^3 at N_c = 1 (40^3 space-time holes; the config's 50^3
# block alone takes minutes to factor): the same ratio of hole, skeleton and fine work per DOF,
# with the rate per DOF extrapolated.  Measured wall times incl. setup on 8 cores: 0.1 / 3 / 40 /
# 8 / 29 s.
CPU_SAMPLE = [
    (0, 0, 10, "full solve (initial guess + 10 iterations) at the config's mesh"),
    (0, 0, 20, "full solve (initial guess + 20 iterations) at the config's mesh"),
    (0, 0, 1, "the config's full 4099^2 mesh: initial guess + 1 iteration timed, the 20-iteration rate extrapolated"),
    (103, 3, 1, "103^3 at N_c=3 (the config's 25^3 holes; the full 259^3 slabs take hours to factor on the host): "
                "initial guess + 1 iteration timed, the 10-iteration rate per DOF extrapolated"),
    (81, 1, 1, "81^3 at N_c=1 (40^3 space-time holes; the config's 50^3 hole block takes minutes to factor on the "
               "host): initial guess + 1 iteration timed, the 10-iteration rate per DOF extrapolated"),
]
CPU_SAMPLE_TIMEOUT_S = 240  # a sample that overruns is reported as unavailable, never waited for
FP64_PEAK_TFLOPS = 37.0  # measured on this pool's B200 (scripts/probe_fp64.cu: DMMA 37.0, DFMA 36.6)
REF_DUMP = os.path.join(ROOT, "oracle", "_ref", "ref_dump")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=int(os.environ.get("ASDSM_BENCH_CONFIG", "1")))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", dest="per_config", action="store_false",
                    help="measure the headline config only")
    ap.add_argument("--only", type=str, default=None, help="comma list of configs for per_config")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
# reference (CPU) side: no import of this package
# ---------------------------------------------------------------------------------------------

def reference_sample(cid, seed):
    """One bounded sample of config `cid` by the compiled reference (oracle/_ref: the reference's
    own sources).  Returns (DOF-iter/s of the K-iteration solve, details).  Context setup
    (factorizations) is excluded, as on the GPU arm (prebuilt plan)."""
    nf, nc, it, what = CPU_SAMPLE[cid]
    with tempfile.TemporaryDirectory() as d:
        prefix = os.path.join(d, "r")
        t0 = time.time()
        subprocess.run([REF_DUMP, "iterate", f"cfg:{cid}:{seed}", str(nf), str(nc), str(it), "0", prefix],
                       stdout=subprocess.DEVNULL, check=True, timeout=CPU_SAMPLE_TIMEOUT_S)
        wall = time.time() - t0
        rows = np.array([[float(x) for x in line.split()] for line in open(prefix + ".hist.txt")
                         if not line.startswith("#")])
        meta = open(prefix + ".meta.txt").read().split("\n")
    fine = [int(x) for x in meta[1].split()]
    coarse = [int(x) for x in meta[2].split()]
    ndof = int(np.prod(fine))
    t_init = rows[0, 6] / 1e3
    t_iter = float(np.mean(rows[1:, 6])) / 1e3 if len(rows) > 1 else 0.0
    k = ITERATIONS[cid]
    t_solve = t_init + k * t_iter  # == the measured total when the sample is the full solve
    return ndof * k / t_solve, {
        "sample_mesh": {"fine_counts": fine, "coarse_counts": coarse, "dof": ndof},
        "iterations_timed": len(rows) - 1, "t_initial_guess_s": t_init, "t_iteration_s": t_iter,
        "t_solve_s_extrapolated" if it != k else "t_solve_s": t_solve, "wall_s_incl_setup": wall}


def run_reference_arm(args):
    """--impl reference: the reference's CPU implementation (oracle/_ref), all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cid = args.config
    if not os.path.exists(REF_DUMP):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_dump not built"}))
        return
    cores = os.cpu_count() or 1
    full = CPU_SAMPLE[cid][2] == ITERATIONS[cid] and CPU_SAMPLE[cid][0] == 0
    for _ in range(args.warmup if full else 0):
        reference_sample(cid, args.seed)
    vals, det = [], None
    for _ in range(args.steps if full else 1):
        v, det = reference_sample(cid, args.seed)
        vals.append(v)
    value = float(np.mean(vals))
    ndof = det["sample_mesh"]["dof"]
    ms = ndof * ITERATIONS[cid] / value * 1e3
    print(json.dumps({
        "impl": "reference", "metric": "fine-grid DOF-iterations/sec", "value": value, "unit": "DOF-iter/s",
        "n_gpus": args.gpus, "steps": len(vals), "warmup": args.warmup if full else 0, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded, BASELINE.json config {cid})",
        "config": config_dict(cid, args.gpus),
        "cpu_baseline": {"value": value, "unit": "DOF-iter/s", "cores": cores, "kind": "reference",
                         "sample": CPU_SAMPLE[cid][3] + "; the reference's own C++ (oracle/_ref) with the "
                                   "Eigen SparseLU stand-in (RCM + band LU), hole solves threaded"},
        "reference_detail": det,
        "e2e": {"value": value, "unit": "DOF-iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------------------------

def ncu_traffic(cid, component, kernels):
    """DRAM bytes per launch (read + write) of `component` at config `cid` from a committed
    `ncu --set full` capture (profiles/r*_traffic*.json, newest round and version first, written
    by scripts/traffic_from_ncu.py), only when every kernel of the capture is one this plan's
    solve graph actually launches; else None."""
    def order(p):
        m = re.match(r"r(\d+)_traffic(?:_v?(\w+))?\.json", os.path.basename(p))
        return (int(m.group(1)), m.group(2) or "") if m else (0, "")
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic*.json")), key=order, reverse=True)

    def norm(n):  # `stencil2d_ym_kernel<1,0>` from either demangler's spelling
        n = n.replace("(anonymous namespace)::", "").replace("asdsm_b200::", "")
        n = re.sub(r"\((?:int|bool)\)", "", n)
        return n.replace(" ", "").replace("false", "0").replace("true", "1")

    def launched(name):
        return any(norm(name) == norm(n) for n in kernels)
    for path in paths:
        try:
            k = json.load(open(path))["kernels"].get(f"{cid}/{component}")
        except Exception:
            continue
        if not k:
            continue
        names = k.get("kernels") or [k["kernel"]]
        if all(launched(n) for n in names):
            return {"bytes": float(k["dram_read_bytes"] + k["dram_write_bytes"]), "kernels": names,
                    "source": os.path.relpath(path, ROOT)}
    return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons (NVML, else nvidia-smi) sampled during the timed region."""

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        # NVML in-process (what nvidia-smi reads) when available: no subprocess spawned inside the
        # timed region; nvidia-smi otherwise
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                    ("sw_power_cap", 0x4)]

            def sample():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = reasons_fn(h)
                return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for _, b in bits]
        except Exception:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")

            def sample():
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                return [x.strip() for x in out.split(",")] if out else None

        def run():
            while not self._stop.is_set():
                try:
                    v = sample()
                    if v:
                        self.samples.append(v)
                except Exception:
                    pass
                self._stop.wait(0.02)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(s[0]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


L2_GBS = [None]  # measured once per run (main)
L2_RESIDENT_BYTES = 64e6  # per-launch working sets below this stay in the 126 MB L2 within a solve


def measure_l2_gbs():
    """L2 bandwidth ceiling for L2-resident kernels: a 32 MB -> 32 MB device copy repeated (the
    64 MB working set stays in the 126 MB L2), read + write bytes over CUDA-event time, best of 5."""
    import torch
    a = torch.ones(4 * 1024 * 1024, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            b.copy_(a)
        e1.record()
        e1.synchronize()
        best = max(best, 20 * 2 * a.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def max_over_ranks(value, device):
    """Max of a per-rank scalar over all ranks (timings: the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# Which components are the north star's HBM-bound fine-grid / merge kernels (>= 60 % target).
HBM_COMPONENTS = ("update_residual", "dots_update", "residual", "skeleton_merge", "merge3d", "gather")


def measure_config(cid, args, world, rank, local, flush, steps, warmup):
    """Value, e2e, per-component rooflines and clocks of config `cid` on this GPU."""
    import torch
    import paper_2303_01163_b200 as pb

    mesh, iters = pb.baseline_mesh(cid)
    prob = pb.baseline_problem(cid, args.seed + rank)  # replicas: independent problems per rank
    t0 = time.time()
    ctx = pb.SolverContext(mesh, prob)
    setup_s = time.time() - t0
    ndof = ctx.fine_size()
    assert [list(mesh.fine_counts), list(mesh.coarse_counts), iters] == [*MESHES[cid], ITERATIONS[cid]]
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=args.seed)
    lib = pb.load_library()
    lib.asdsm_plan_stream.restype = ctypes.c_void_p
    lib.asdsm_plan_stream.argtypes = [ctypes.c_void_p]
    stream = torch.cuda.Stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    copt = opts._c()

    def flush_l2(s):
        with torch.cuda.stream(s):
            flush.fill_(1.0)

    def step():
        pb.asdsm._check(lib.asdsm_iterate_async(ctx._h, ctypes.byref(copt), sp))

    for _ in range(max(warmup, 0)):
        flush_l2(stream)
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        flush_l2(stream)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = ctx.launch_count()
    kernels = ctx.kernels()
    ms = max_over_ranks(float(np.mean(times)), "cuda")
    value = world * ndof * iters / (ms / 1e3)

    hist = np.empty((iters + 1) * 7)
    nrec, stop = ctypes.c_int(), ctypes.c_int()
    pb.asdsm._check(lib.asdsm_fetch(ctx._h, sp, pb.asdsm._dptr(hist), ctypes.byref(nrec), ctypes.byref(stop),
                                    None, None))
    res = hist[: nrec.value * 7].reshape(-1, 7)[:, 1]

    # ---- component roofline (CUDA events on the launching stream, inside this run)
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    n = 16
    names = ctypes.create_string_buffer(64 * n)
    cms, cby, cfl = (ctypes.c_double * n)(), (ctypes.c_double * n)(), (ctypes.c_double * n)()
    cps, cnt = (ctypes.c_int * n)(), ctypes.c_int()
    lib.asdsm_profile_components.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    pb.asdsm._check(lib.asdsm_profile_components(ctx._h, sp, 10, n, names, cms, cby, cfl, cps, ctypes.byref(cnt)))
    comps = []
    for i in range(cnt.value):
        nm = names.raw[64 * i:64 * i + 64].split(b"\0")[0].decode()
        c = {"name": nm, "ms_per_launch": cms[i], "launches_per_solve": cps[i],
             "share_of_step": cms[i] * cps[i] / ms, "bytes_per_launch": cby[i], "flops_per_launch": cfl[i],
             "gbs": cby[i] / (cms[i] / 1e3) / 1e9 if cms[i] > 0 else None,
             "tflops": cfl[i] / (cms[i] / 1e3) / 1e12 if cms[i] > 0 and cfl[i] > 0 else None}
        comps.append(c)

    def roof_of(c):
        share = c["ms_per_launch"] * c["launches_per_solve"] / ms
        if c["flops_per_launch"] > 0 and c["flops_per_launch"] / max(c["bytes_per_launch"], 1) > FP64_PEAK_TFLOPS * 1e3 / hbm:
            ach = c["flops_per_launch"] / (c["ms_per_launch"] / 1e3) / 1e12
            tr = ncu_traffic(cid, c["name"], kernels)
            return {"kernel": c["name"], "bound": "tensor", "achieved": ach, "peak": FP64_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": ach / FP64_PEAK_TFLOPS, "traffic": tr["bytes"] if tr else None,
                    "traffic_source": tr, "share_of_step": share,
                    "peak_source": "fp64 DMMA/DFMA peak measured with scripts/probe_fp64.cu (MEASURED_PEAKS has no "
                                   "fp64); flops are dense-equivalent (the even/odd split executes half)"}
        if c["bytes_per_launch"] < 1e6:
            return {"kernel": c["name"], "bound": "latency", "achieved": None, "peak": None, "unit": None,
                    "frac": None, "traffic": None, "share_of_step": share,
                    "note": "under 1 MB per launch on a handful of SMs: dependency-chain latency, not bandwidth"}
        ach = c["bytes_per_launch"] / (c["ms_per_launch"] / 1e3) / 1e9
        tr = ncu_traffic(cid, c["name"], kernels)
        out = {"kernel": c["name"], "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
               "frac": ach / hbm, "traffic": tr["bytes"] if tr else None,
               "traffic_source": tr, "share_of_step": share,
               "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
        if l2_gbs and c["bytes_per_launch"] < L2_RESIDENT_BYTES:
            # the kernel's arrays fit the 126 MB L2 and stay resident between the solve's launches:
            # its ceiling is the L2 bandwidth (measured in this run), not HBM
            out["l2"] = {"peak": l2_gbs, "unit": "GB/s", "frac": ach / l2_gbs,
                         "peak_source": "this run: 64 MB L2-resident device copy (measure_l2_gbs)"}
        return out

    l2_gbs = L2_GBS[0]
    cand = [c for c in comps if c["launches_per_solve"] > 0]
    dom = max(cand, key=lambda c: c["ms_per_launch"] * c["launches_per_solve"])
    roof_all = [roof_of(c) for c in cand]
    roof_hbm = [r for r in roof_all if r["kernel"] in HBM_COMPONENTS]

    # ---- e2e through the C-ABI with pinned host buffers
    b = ctx.bundle
    h_fine = torch.from_numpy(b["fine"]).pin_memory()
    h_slab = [torch.from_numpy(x).pin_memory() for x in b["aniso"]]
    h_coarse = torch.from_numpy(b["coarse"]).pin_memory()
    h_exact = torch.from_numpy(ctx.exact).pin_memory() if ctx.exact is not None else None
    h_u = torch.empty(ndof, dtype=torch.float64).pin_memory()
    h_r = torch.empty(ndof, dtype=torch.float64).pin_memory()
    h_hist = torch.empty((iters + 1) * 7, dtype=torch.float64).pin_memory()
    dp = lambda t: ctypes.cast(ctypes.c_void_p(t.data_ptr()), ctypes.POINTER(ctypes.c_double))  # noqa: E731
    slabs = (ctypes.POINTER(ctypes.c_double) * 3)()
    for a, x in enumerate(h_slab):
        slabs[a] = dp(x)
    pstream = torch.cuda.ExternalStream(lib.asdsm_plan_stream(ctx._h))

    def e2e_step():
        # asdsm_solve: this step's right-hand sides up, the solve, history + u + r down; one sync
        pb.asdsm._check(lib.asdsm_solve(ctx._h, dp(h_fine), slabs, dp(h_coarse),
                                        dp(h_exact) if h_exact is not None else None, ctypes.byref(copt),
                                        dp(h_hist), ctypes.byref(nrec), ctypes.byref(stop), dp(h_u), dp(h_r)))

    for _ in range(max(warmup, 3)):
        flush_l2(pstream)
        e2e_step()
    etimes = []
    for _ in range(max(steps, 5)):
        flush_l2(pstream)
        a = torch.cuda.Event(enable_timing=True)
        bb = torch.cuda.Event(enable_timing=True)
        a.record(pstream)
        e2e_step()
        bb.record(pstream)
        bb.synchronize()
        etimes.append(a.elapsed_time(bb))
    ems = max_over_ranks(float(np.mean(etimes)), "cuda")
    h2d = 8 * (b["fine"].size + sum(x.size for x in b["aniso"]) + b["coarse"].size + (ndof if h_exact is not None else 0))
    d2h = 8 * (2 * ndof + (iters + 1) * 7)
    e2e = {"value": world * ndof * iters / (ems / 1e3), "unit": "DOF-iter/s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "ms_per_step": ems, "steps": len(etimes),
           "ms_all": [round(t, 4) for t in etimes]}
    if not np.isfinite(h_u.numpy()).all():
        raise RuntimeError("non-finite solution")

    out = {
        "value": value, "ms_per_step": ms, "steps": steps, "warmup": warmup,
        "config": config_dict(cid, world),
        "e2e": e2e, "roofline": roof_of(dom), "roofline_hbm": roof_hbm, "roofline_components": roof_all,
        "gpu_launches": launches, "kernels": kernels, "clocks": clocks, "components": comps, "setup_s": setup_s,
        "res_l2_first_last": [float(res[0]), float(res[-1])], "step_ms_all": times,
    }
    del ctx
    torch.cuda.synchronize()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    sys.path.insert(0, ROOT)
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    L2_GBS[0] = measure_l2_gbs()

    cid = args.config
    head = measure_config(cid, args, world, rank, local, flush, args.steps, args.warmup)
    per = {}
    if args.per_config and world == 1:
        only = [int(x) for x in args.only.split(",")] if args.only else range(len(CONFIG_NAMES))
        for c in only:
            t0 = time.time()
            per[c] = head if c == cid else measure_config(c, args, world, rank, local, flush,
                                                          max(3, min(args.steps, 5)), max(args.warmup, 3))
            print(f"[bench] config {c}: {per[c]['ms_per_step']:.3f} ms/solve, setup {per[c]['setup_s']:.1f} s, "
                  f"measured in {time.time() - t0:.1f} s", file=sys.stderr, flush=True)

    # ---- CPU baseline: the compiled reference on this box's host cores (rank 0, N=1), after
    # every GPU measurement (nothing else runs on the host while it is timed)
    cpu = {}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(REF_DUMP):
        for c in ([cid] + [c for c in per if c != cid]):
            t0 = time.time()
            try:
                v, det = reference_sample(c, args.seed)
            except subprocess.TimeoutExpired:
                cpu[c] = {"unavailable": f"reference sample exceeded {CPU_SAMPLE_TIMEOUT_S} s on this host"}
                continue
            print(f"[bench] cpu sample config {c}: {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
            cpu[c] = {"value": v, "unit": "DOF-iter/s", "cores": os.cpu_count(), "kind": "reference",
                      "sample": CPU_SAMPLE[c][3] + "; the reference's own C++ (oracle/_ref, Eigen SparseLU stand-in: "
                                "RCM + band LU), hole solves threaded, context setup excluded", "detail": det}

    line = {
        "metric": "fine-grid DOF-iterations/sec",
        "value": head["value"],
        "unit": "DOF-iter/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic (seeded, BASELINE.json config {cid})",
        "config": head["config"],
        "e2e": head["e2e"],
        "roofline": head["roofline"],
        "roofline_hbm": head["roofline_hbm"],
        "roofline_components": head["roofline_components"],
        "cpu_baseline": cpu.get(cid),
        "gpu_launches": head["gpu_launches"],
        "clocks": head["clocks"],
        "l2_gbs_measured": L2_GBS[0],
        "kernels": head["kernels"],
        "components": head["components"],
        "setup_s": head["setup_s"],
        "res_l2_first_last": head["res_l2_first_last"],
        "step_ms_all": head["step_ms_all"],
    }
    if per:
        pc = []
        for c, r in per.items():
            e = {k: r[k] for k in ("config", "value", "ms_per_step", "steps", "warmup", "e2e", "roofline",
                                   "roofline_hbm", "gpu_launches", "clocks", "res_l2_first_last")}
            e["e2e"] = {k: v for k, v in e["e2e"].items() if k != "ms_all"}
            e["cpu_baseline"] = cpu.get(c)
            if c != cid:
                e["roofline_components"] = r["roofline_components"]
            pc.append(e)
        line["per_config"] = pc
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
