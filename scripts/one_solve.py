"""One warm ASDSM solve of a BASELINE config on cuda:0 (for ncu launch lists):
python scripts/one_solve.py CONFIG [SOLVES]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2303_01163_b200 as pb  # noqa: E402

cid = int(sys.argv[1])
nsolve = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mesh, iters = pb.baseline_mesh(cid)
ctx = pb.SolverContext(mesh, pb.baseline_problem(cid, 0))
lib = pb.load_library()
opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=0)._c()
s = torch.cuda.Stream()
for _ in range(nsolve):
    pb.asdsm._check(lib.asdsm_iterate_async(ctx._h, ctypes.byref(opts), ctypes.c_void_p(s.cuda_stream)))
torch.cuda.synchronize()
print("launches per solve", ctx.launch_count())
