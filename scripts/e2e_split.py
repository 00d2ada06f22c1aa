"""Where the e2e time goes (config 1): device-timed pieces of asdsm_solve on the plan stream."""
import ctypes, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2303_01163_b200 as pb
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mesh, iters = pb.baseline_mesh(cid)
ctx = pb.SolverContext(mesh, pb.baseline_problem(cid, 0))
opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=0)
st0 = ctx.iterate(opts)
bun = {k: ([2.0 * x for x in v] if k == "aniso" else 2.0 * v) for k, v in ctx.bundle.items()}
st2 = ctx.solve(bun, None, opts)
print("u x2", np.array_equal(st2.u, 2 * st0.u), "r x2", np.array_equal(st2.r, 2 * st0.r))
print("s0", [h.s_hat for h in st0.history][:6]); print("s2", [h.s_hat for h in st2.history][:6])
lib = pb.load_library()
lib.asdsm_plan_stream.restype = ctypes.c_void_p
n = ctx.fine_size()
b = ctx.bundle
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
h_fine, h_coarse = pin(b["fine"]), pin(b["coarse"]); h_slab = [pin(x) for x in b["aniso"]]
h_u = torch.empty(n, dtype=torch.float64).pin_memory(); h_r = torch.empty(n, dtype=torch.float64).pin_memory()
h_hist = torch.empty((iters + 1) * 7, dtype=torch.float64).pin_memory()
dp = lambda t: ctypes.cast(ctypes.c_void_p(t.data_ptr()), ctypes.POINTER(ctypes.c_double))
slabs = (ctypes.POINTER(ctypes.c_double) * 3)()
for a, x in enumerate(h_slab): slabs[a] = dp(x)
copt = opts._c(); nrec, stop = ctypes.c_int(), ctypes.c_int()
ps = torch.cuda.ExternalStream(lib.asdsm_plan_stream(ctx._h))
sp = ctypes.c_void_p(lib.asdsm_plan_stream(ctx._h))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
def timed(fn, reps=10, label="", fl=False):
    fn(); torch.cuda.synchronize()
    ts, walls = [], []
    for _ in range(reps):
        if fl:
            with torch.cuda.stream(ps): flush.fill_(1.0)
        a = torch.cuda.Event(enable_timing=True); bb = torch.cuda.Event(enable_timing=True)
        w = time.perf_counter(); a.record(ps); fn(); bb.record(ps); bb.synchronize(); walls.append(time.perf_counter() - w)
        ts.append(a.elapsed_time(bb))
    print(f"{label:40s} device {np.mean(ts)*1e3:8.1f} us  wall {np.mean(walls)*1e6:8.1f} us")
timed(lambda: pb.asdsm._check(lib.asdsm_set_bundle(ctx._h, dp(h_fine), slabs, dp(h_coarse), None, 0)), label="set_bundle (sync)")
timed(lambda: pb.asdsm._check(lib.asdsm_iterate_async(ctx._h, ctypes.byref(copt), sp)), label="iterate_async")
timed(lambda: pb.asdsm._check(lib.asdsm_fetch(ctx._h, sp, dp(h_hist), ctypes.byref(nrec), ctypes.byref(stop), dp(h_u), dp(h_r))), label="fetch u,r")
timed(lambda: pb.asdsm._check(lib.asdsm_fetch(ctx._h, sp, dp(h_hist), ctypes.byref(nrec), ctypes.byref(stop), None, None)), label="fetch hist only")
timed(lambda: pb.asdsm._check(lib.asdsm_solve(ctx._h, dp(h_fine), slabs, dp(h_coarse), None, ctypes.byref(copt), dp(h_hist), ctypes.byref(nrec), ctypes.byref(stop), dp(h_u), dp(h_r))), label="asdsm_solve")
timed(lambda: pb.asdsm._check(lib.asdsm_solve(ctx._h, dp(h_fine), slabs, dp(h_coarse), None, ctypes.byref(copt), dp(h_hist), ctypes.byref(nrec), ctypes.byref(stop), dp(h_u), dp(h_r))), label="asdsm_solve, L2 flushed", fl=True)
timed(lambda: pb.asdsm._check(lib.asdsm_iterate_async(ctx._h, ctypes.byref(copt), sp)), label="iterate_async, L2 flushed", fl=True)
dfine = torch.empty(n, dtype=torch.float64, device="cuda")
def tcopy():
    with torch.cuda.stream(ps): dfine.copy_(h_fine, non_blocking=True)
timed(tcopy, label="torch H2D of h_fine")
def tcopy2():
    with torch.cuda.stream(ps): h_u.copy_(dfine, non_blocking=True)
timed(tcopy2, label="torch D2H into h_u")
hf2 = torch.empty(n, dtype=torch.float64).pin_memory(); hf2.copy_(h_fine)
timed(lambda: pb.asdsm._check(lib.asdsm_set_bundle(ctx._h, dp(hf2), slabs, dp(h_coarse), None, 0)), label="set_bundle (sync) fresh pinned")
os.environ["ASDSM_DEBUG_PTR"] = "1"
pb.asdsm._check(lib.asdsm_set_bundle(ctx._h, dp(h_fine), slabs, dp(h_coarse), None, 0))
pb.asdsm._check(lib.asdsm_set_bundle(ctx._h, dp(hf2), slabs, dp(h_coarse), None, 0))
del os.environ["ASDSM_DEBUG_PTR"]
for r in range(3):
    timed(tcopy, label="torch H2D of h_fine")
    timed(lambda: pb.asdsm._check(lib.asdsm_set_bundle(ctx._h, dp(h_fine), slabs, dp(h_coarse), None, 0)), label="set_bundle (sync) again")
torch.cuda.synchronize()
os._exit(0)
