"""Per-iteration GPU vs reference residual history with the reference's own ordering spread
(diagnostic for the parity bound): python scripts/diag_history.py SPEC NF NC ITERS SEED"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_01163_b200 as pb  # noqa: E402
from ref_tools import ref_iterate_pair  # noqa: E402
from test_gpu_parity import _ctx  # noqa: E402

spec, nf, nc, iters, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
ref, (alt, nat) = ref_iterate_pair(spec, nf, nc, iters, seed)
ctx, mesh, _ = _ctx(spec, nf, nc)
st = ctx.iterate(pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=seed))
got = np.array([h.res_l2 for h in st.history])
sg = np.array([h.s_hat for h in st.history])
want, walt = ref["hist"][:, 1], alt["hist"][:, 1]
print("env:", {k: v for k, v in os.environ.items() if k.startswith("ASDSM_")})
print(" k   gpu-ref rel   alt-ref rel   s_gpu/s_ref-1   s_alt/s_ref-1")
for k in range(len(want)):
    print(f"{k:2d}  {(got[k]-want[k])/want[k]:+.3e}  {(walt[k]-want[k])/want[k]:+.3e}  "
          f"{(sg[k]/ref['hist'][k,5]-1) if k else 0:+.3e}  {(alt['hist'][k,5]/ref['hist'][k,5]-1) if k else 0:+.3e}")
sc = np.max(np.abs(ref["u"]))
print(f"u: gpu-ref {np.max(np.abs(st.u-ref['u']))/sc:.3e}  alt-ref {np.max(np.abs(alt['u']-ref['u']))/sc:.3e}")
