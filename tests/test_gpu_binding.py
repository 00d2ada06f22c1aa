"""The reference-side binding of INTEGRATION.md, compiled against the reference's own headers and
library (tests/cxx/ref_binding.cpp, built into oracle/_ref by oracle/Makefile): the reference's
asdsm_iterate(ProblemSpec, MeshConfig, IterateOptions) (solver.hpp:160-161) against
asdsm_iterate_b200 with the same arguments -- caller-defined ProblemSpec fields as C callbacks,
the IterateOptions observer through asdsm_iterate_observed.

Cases: a catalogue example (constant and variable coefficients), a variable-coefficient problem
outside the catalogue, and advection-dominated problems (cell Peclet number up to 10 on the fine
step: complex modes on every axis).  Bound as test_gpu_parity: final u within relative 1e-10,
residual history within max(1e-10, 10x the reference's own fill-ordering spread).
"""
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_binding")

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/ref_binding not built")]


def _hist(path):
    rows = [list(map(float, ln.split())) for ln in open(path) if not ln.startswith("#")]
    return np.array(rows)


def _run(case, nf, nc, iters, seed, env=None):
    with tempfile.TemporaryDirectory() as d:
        prefix = os.path.join(d, "o")
        e = dict(os.environ)
        e.update(env or {})
        p = subprocess.run([BIN, case, str(nf), str(nc), str(iters), str(seed), prefix], env=e, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr
        out = {k: _hist(f"{prefix}.{k}.hist.txt") for k in ("ref", "gpu")}
        out.update({f"u_{k}": np.fromfile(f"{prefix}.{k}.u.f64") for k in ("ref", "gpu")})
        out["obs"] = np.array([list(map(float, ln.split())) for ln in open(prefix + ".obs.txt")])
    return out


@pytest.mark.parametrize("case,nf,nc,iters,seed", [
    ("ex:1:1", 99, 9, 10, 0),
    ("ex:1:2", 49, 4, 8, 1),
    ("var", 49, 4, 8, 2),
    ("adv:0.01", 99, 9, 10, 3),
    ("adv:0.001", 99, 9, 10, 4),
    # cell Peclet 5 / 2.5 on holes of 49 and 99 points: no stable eigenvector scaling on either
    # axis, so the separable solvers cannot take these boxes -- the plan falls back to the
    # block-Thomas path with the same constant operator (Solver::init)
    ("adv:0.001", 199, 3, 8, 5),
    ("adv:0.001", 199, 1, 6, 6),
])
def test_reference_binding_matches_reference(case, nf, nc, iters, seed):
    a = _run(case, nf, nc, iters, seed)
    alt = _run(case, nf, nc, iters, seed, {"ASDSM_STUB_ORDER": "cm"})  # the reference's ordering spread
    ref, gpu = a["ref"][:, 1], a["gpu"][:, 1]
    assert len(ref) == len(gpu) == iters + 1
    spread = np.maximum.accumulate(np.abs(alt["ref"][:, 1] - ref) / ref)
    tol = ref * np.maximum(1e-10, 10.0 * spread)
    rel = np.abs(gpu - ref) / ref
    assert np.all(np.abs(gpu - ref) <= tol), (rel, tol / ref)
    assert np.array_equal(a["gpu"][:, 5] == 0.0, a["ref"][:, 5] == 0.0)  # accept / revert decisions
    urel = np.max(np.abs(a["u_gpu"] - a["u_ref"])) / np.max(np.abs(a["u_ref"]))
    assert urel < 1e-10, urel
    # the observer saw every record, k = 0 first, with the record's values
    assert np.array_equal(a["obs"][:, 0], np.arange(iters + 1))
    assert np.array_equal(a["obs"][:, 1], gpu)
    print(f"{case}: history max rel {rel.max():.2e}, u max rel {urel:.2e}")
