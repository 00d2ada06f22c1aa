"""ASDSM benchmark on B200.

Metric: fine-grid DOF-iterations/s = (fine unknowns x ASDSM iterations) / solve time.  One
"step" = one full ASDSM solve of the configured BASELINE.json problem (initial guess + K
iterations, K from BASELINE.json), on a prebuilt plan (the reference's SolverContext: tables,
operators) with the assembled right-hand-side bundle resident in HBM; L2 flushed between
steps.  `e2e`: the same solve through the C-ABI with pinned HOST buffers (H2D of the bundle,
D2H of u, r and the history inside the timed region).

  python bench.py [--config 1] [--steps K] [--warmup W] [--gpus N] [--impl ours|reference]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_NAMES = [
    "2d_steady_N128_manufactured",
    "2d_steady_N1024_bumps8",
    "2d_advection_N4096_bumps16",
    "3d_steady_N256_manufactured",
    "2d_time_N512_spacetime_bumps8",
]
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
    ap.add_argument("--no-all-configs", dest="all_configs", action="store_false",
                    help="skip timing every other BASELINE config (value only)")
    return ap.parse_args()


def ncu_traffic(cid, kernel):
    """DRAM bytes per launch (read + write) of `kernel` at config `cid` from the committed ncu
    --set full capture (profiles/r*_traffic.json, newest round first), else None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        try:
            k = json.load(open(path))["kernels"].get(f"{cid}/{kernel}")
        except Exception:
            continue
        if k:
            return float(k["dram_read_bytes"] + k["dram_write_bytes"])
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


def max_over_ranks(value, device):
    """Max of a per-rank scalar over all ranks (timings: the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reference_solve(cid, seed, iters):
    """One solve of the compiled reference (oracle/_ref: the reference's own sources); returns
    (solve seconds excluding context setup, history rows)."""
    with tempfile.TemporaryDirectory() as d:
        prefix = os.path.join(d, "r")
        subprocess.check_call([REF_DUMP, "iterate", f"cfg:{cid}:{seed}", "0", "0", str(iters), "0", prefix],
                              stdout=subprocess.DEVNULL)
        rows = np.array([[float(x) for x in line.split()] for line in open(prefix + ".hist.txt") if not line.startswith("#")])
    return float(rows[:, 6].sum()) / 1e3, rows


def run_reference_arm(args):
    """--impl reference: the reference's CPU implementation (oracle/_ref), all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2303_01163_b200 as pb
    cid = args.config
    mesh, iters = pb.baseline_mesh(cid)
    ndof = mesh.point_count(pb.MeshKind.fine(mesh.dim))
    cores = os.cpu_count() or 1
    if not os.path.exists(REF_DUMP):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_dump not built"}))
        return
    # bounded sample: full solves for the small configs, (initial guess + 1 iteration) beyond
    sample_iters = iters if ndof <= 2_000_000 else 1
    for _ in range(args.warmup if sample_iters == iters else 0):
        reference_solve(cid, args.seed, sample_iters)
    times = []
    for _ in range(args.steps if sample_iters == iters else 1):
        t, rows = reference_solve(cid, args.seed, sample_iters)
        times.append(t)
    t = float(np.mean(times))
    value = ndof * sample_iters / t
    sample = (f"full solve ({iters} iterations + initial guess), context setup excluded"
              if sample_iters == iters else "initial guess + 1 iteration, context setup excluded")
    print(json.dumps({
        "impl": "reference", "metric": "fine-grid DOF-iterations/sec", "value": value, "unit": "DOF-iter/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded, BASELINE.json config {cid})",
        "config": {"workload": CONFIG_NAMES[cid], "config_id": cid, "fine_counts": mesh.fine_counts,
                   "coarse_counts": mesh.coarse_counts, "iterations": iters, "dof": ndof},
        "cpu_baseline": {"value": value, "unit": "DOF-iter/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "DOF-iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch
    import paper_2303_01163_b200 as pb

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")

    cid = args.config
    mesh, iters = pb.baseline_mesh(cid)
    prob = pb.baseline_problem(cid, args.seed + rank)  # replicas: independent problems per rank
    t0 = time.time()
    ctx = pb.SolverContext(mesh, prob)
    setup_s = time.time() - t0
    ndof = ctx.fine_size()
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=args.seed)
    lib = pb.load_library()
    lib.asdsm_plan_stream.restype = ctypes.c_void_p
    lib.asdsm_plan_stream.argtypes = [ctypes.c_void_p]
    stream = torch.cuda.Stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    copt = opts._c()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush_l2(s):
        with torch.cuda.stream(s):
            flush.fill_(1.0)

    def step():
        pb.asdsm._check(lib.asdsm_iterate_async(ctx._h, ctypes.byref(copt), sp))

    for _ in range(max(args.warmup, 0)):
        flush_l2(stream)
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
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
    # Rooflines.  The headline object is the fine-grid residual/update pass (north-star kernels 1
    # and 4, the HBM-bound pass the >= 60 % target is stated for); every component gets its own
    # entry in roofline_components, and the dominant kernel of the step is named with its bound
    # (kernels that move < 1 MB per launch and do no GEMM work are latency bound: no roofline).
    def roof_of(c):
        if c["flops_per_launch"] > 0 and c["flops_per_launch"] / max(c["bytes_per_launch"], 1) > FP64_PEAK_TFLOPS * 1e3 / hbm:
            ach = c["flops_per_launch"] / (c["ms_per_launch"] / 1e3) / 1e12
            return {"kernel": c["name"], "bound": "tensor", "achieved": ach, "peak": FP64_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": ach / FP64_PEAK_TFLOPS, "traffic": None,
                    "peak_source": "fp64 DMMA/DFMA peak measured with scripts/probe_fp64.cu (MEASURED_PEAKS has no fp64)"}
        if c["bytes_per_launch"] < 1e6:
            return {"kernel": c["name"], "bound": "latency", "achieved": None, "peak": None, "unit": None,
                    "frac": None, "traffic": None,
                    "note": "under 1 MB per launch on a handful of SMs: dependency-chain latency, not bandwidth"}
        ach = c["bytes_per_launch"] / (c["ms_per_launch"] / 1e3) / 1e9
        return {"kernel": c["name"], "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": ncu_traffic(cid, c["name"]), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}

    cand = [c for c in comps if c["name"] not in ("step_dots_overhead",)]
    # the fine-grid update pass as the step runs it: fused with the step dots where it applies
    upd = next((c for c in comps if c["name"] == "dots_update"),
               next((c for c in comps if c["name"] == "update_residual"), cand[0]))
    roof = roof_of(upd)
    roof["share_of_step"] = upd["ms_per_launch"] * upd["launches_per_solve"] / ms
    dom = max(cand, key=lambda c: c["ms_per_launch"] * c["launches_per_solve"])
    roof_dom = roof_of(dom)
    roof_dom["share_of_step"] = dom["ms_per_launch"] * dom["launches_per_solve"] / ms
    roof_all = []
    for c in cand:
        r = roof_of(c)
        roof_all.append({"kernel": c["name"], "bound": r["bound"], "achieved": r["achieved"], "unit": r["unit"],
                         "frac": r["frac"], "share_of_step": c["ms_per_launch"] * c["launches_per_solve"] / ms})

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

    for _ in range(max(args.warmup, 5)):
        flush_l2(pstream)
        e2e_step()
    etimes = []
    for _ in range(max(args.steps, 10)):
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
    assert np.allclose(h_u.numpy(), h_u.numpy())  # touch the result

    # ---- CPU baseline: the compiled reference on this box's host cores (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(REF_DUMP) and ndof <= 2_000_000:
        tcpu, _ = reference_solve(cid, args.seed, iters)
        cpu = {"value": ndof * iters / tcpu, "unit": "DOF-iter/s", "cores": os.cpu_count(), "kind": "reference",
               "sample": f"one full solve ({iters} iterations + initial guess) of the same problem by the reference's "
                         "own code (oracle/_ref, Eigen stand-in), hole solves on all host threads, setup excluded",
               "seconds": tcpu}

    line = {
        "metric": "fine-grid DOF-iterations/sec",
        "value": value,
        "unit": "DOF-iter/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic (seeded, BASELINE.json config {cid})",
        "config": {"workload": CONFIG_NAMES[cid], "config_id": cid, "fine_counts": mesh.fine_counts,
                   "coarse_counts": mesh.coarse_counts, "iterations": iters, "dof": ndof,
                   "l2": "flushed between steps (256 MB write)",
                   "parallelism": f"replicas x{world}" if world > 1 else "1gpu"},
        "e2e": e2e,
        "roofline": roof,
        "roofline_dominant": roof_dom,
        "roofline_components": roof_all,
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clocks,
        "components": comps,
        "setup_s": setup_s,
        "res_l2_first_last": [float(res[0]), float(res[-1])],
        "step_ms_all": times,
    }
    if args.all_configs and rank == 0:
        others = {}
        for c2 in range(len(CONFIG_NAMES)):
            m2, it2 = pb.baseline_mesh(c2)
            ctx2 = pb.SolverContext(m2, pb.baseline_problem(c2, args.seed))
            o2 = pb.IterateOptions(tol=0.0, max_iter=it2, stagnation_window=0, rng_seed=args.seed)._c()
            for _ in range(2):
                pb.asdsm._check(lib.asdsm_iterate_async(ctx2._h, ctypes.byref(o2), sp))
            torch.cuda.synchronize()
            tt = []
            for _ in range(3):
                flush_l2(stream)
                a = torch.cuda.Event(enable_timing=True)
                bb = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                pb.asdsm._check(lib.asdsm_iterate_async(ctx2._h, ctypes.byref(o2), sp))
                bb.record(stream)
                bb.synchronize()
                tt.append(a.elapsed_time(bb))
            m_ = float(np.mean(tt))
            others[CONFIG_NAMES[c2]] = {"ms_per_step": m_, "value": ctx2.fine_size() * it2 / (m_ / 1e3),
                                        "dof": ctx2.fine_size(), "iterations": it2}
            del ctx2
        line["all_configs"] = others
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
