"""Stage-by-stage GPU vs reference error (initial guess, one error guess, final u) with the
reference's own CM-ordering spread beside it: python scripts/diag_stages.py SPEC NF NC ITERS SEED"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_01163_b200 as pb  # noqa: E402
from ref_tools import ref_error_guess, ref_iterate_pair  # noqa: E402
from test_gpu_parity import _ctx  # noqa: E402

spec, nf, nc, iters, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
ref, (alt,) = ref_iterate_pair(spec, nf, nc, iters, seed, orders=("cm",))
ctx, mesh, _ = _ctx(spec, nf, nc)


def rep(name, got, want, other):
    sc = np.max(np.abs(want))
    d = np.abs(got - want)
    i = int(np.argmax(d))
    idx = np.unravel_index(i, tuple(reversed(mesh.fine_counts)))[::-1]
    print(f"{name}: gpu {d[i] / sc:.3e} at {idx} (|want| there {abs(want[i]) / sc:.2e}),  "
          f"cm-order {np.max(np.abs(other - want)) / sc:.3e},  gpu l2-rel {np.linalg.norm(got - want) / np.linalg.norm(want):.3e}")


u0 = ctx.initial_guess()
rep("u0", u0, ref["u0"], alt["u0"])
e_ref, s_ref = ref_error_guess(spec, nf, nc, 7, ref["r0"])
e = ctx.error_guess(ref["r0"], 7)
rep("e(r0)", e, e_ref, e_ref)
st = ctx.iterate(pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=seed))
rep("u_final", st.u, ref["u"], alt["u"])
