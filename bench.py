"""ASDSM benchmark on B200.

Metric: fine-grid DOF-iterations/s = (fine unknowns x ASDSM iterations) / solve time, one
"step" = one full ASDSM solve (initial guess + K iterations, BASELINE.json's count) of the
configured problem, inputs (the assembled right-hand-side bundle) resident in HBM.
`e2e`: the same solve through the C-ABI with HOST buffers (H2D of the bundle, D2H of the
solution and history inside the timed region).

  python bench.py [--config 1] [--steps K] [--warmup W] [--gpus N] [--impl ours|reference]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=int(os.environ.get("ASDSM_BENCH_CONFIG", "1")))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self):
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def main():
    args = parse()
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
    prob = pb.baseline_problem(cid, args.seed + rank)
    t0 = time.time()
    ctx = pb.SolverContext(mesh, prob)
    setup_s = time.time() - t0
    ndof = ctx.fine_size()
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=args.seed)
    lib = pb.load_library()
    stream = torch.cuda.Stream()  # dedicated stream: events and the solve share it
    sp = ctypes.c_void_p(stream.cuda_stream)
    copt = opts._c()

    # L2 flush buffer (> 126 MB L2) written between timed steps.
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step():
        pb.asdsm._check(lib.asdsm_iterate_async(ctx._h, ctypes.byref(copt), sp))

    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    times = []
    sampler = ClockSampler()
    sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
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
    ms = float(np.mean(times))
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = world * ndof * iters / (ms / 1e3)

    # history sanity
    hist = np.empty((iters + 1) * 7)
    nrec, stop = ctypes.c_int(), ctypes.c_int()
    pb.asdsm._check(lib.asdsm_fetch(ctx._h, sp, pb.asdsm._dptr(hist), ctypes.byref(nrec), ctypes.byref(stop), None, None))
    res = hist[: nrec.value * 7].reshape(-1, 7)[:, 1]

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
        "data": "synthetic (seeded, BASELINE.json config %d)" % cid,
        "config": {"workload": CONFIG_NAMES[cid], "config_id": cid, "fine_counts": mesh.fine_counts,
                   "coarse_counts": mesh.coarse_counts, "iterations": iters, "dof": ndof,
                   "l2": "flushed between steps (256 MB write)", "parallelism": "replicas" if world > 1 else "1gpu"},
        "gpu_launches": launches,
        "clocks": clocks,
        "setup_s": setup_s,
        "res_l2_first_last": [float(res[0]), float(res[-1])],
        "step_ms_all": times,
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
