"""CPU suite: the oracle restatement pinned against the reference's own outputs.

(1) golden vectors written by the reference's own sources (tests/golden, make_golden.py);
(2) the figures the reference's acceptance run recorded (proj/test_output.txt), 3 s.f.
Tolerances as in test_gpu_parity.py.
"""
import glob
import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import asdsm_oracle as O  # noqa: E402

GOLD = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz")))

COEFFS = {  # constant coefficients of the problems in the goldens (problems.cpp, asdsm_problems.hpp)
    "ex:1:1": ([1, 1], [1, 1]), "ex:3:1": ([1], [1]), "ex:4:1": ([1, 1, 1], [1, 1, 1]),
    "cfg:0": ([1, 1], [1, 1]), "cfg:1": ([0.1, 0.1], [1.0, -0.5]), "cfg:2": ([0.01, 0.01], [1.0, 1.0]),
    "cfg:3": ([1, 1, 1], [0.5, 0.5, 0.5]), "cfg:4": ([0.5, 0.5], [1.0, 0.0]),
}


def eval_floor(A, u):
    absau = abs(A) @ np.abs(u)
    return np.finfo(np.float64).eps * float(np.linalg.norm(absau))


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[:-4] for p in GOLD])
def test_oracle_matches_reference_goldens(path):
    g = np.load(path)
    spec = str(g["spec"])
    key = spec if spec.startswith("ex") else ":".join(spec.split(":")[:2])
    alpha, beta = COEFFS[key]
    dim, ta = int(g["dim"]), int(g["time_axis"])
    mesh = O.Mesh.create(dim, list(g["fine"]), list(g["coarse"]), ta)
    prob = O.constant_problem(dim, alpha, beta, ta >= 0)
    bundle = {"fine": g["b_fine"], "aniso": [g[f"b_slab{a}"] for a in range(dim)], "coarse": g["b_coarse"]}
    exact = g["exact"] if g["exact"].size else None
    u, r, hist, stop = O.asdsm_iterate(mesh, prob, int(g["iters"]), int(g["seed"]), exact=exact, bundle=bundle)
    want = g["hist"][:, 1]
    got = np.array([h.res_l2 for h in hist])
    spread = np.maximum.accumulate(np.abs(g["hist_cm"][:, 1] - want) / want)
    A = O.assemble_operator(mesh, prob, 0)
    tol = np.maximum(want * np.maximum(1e-10, 10 * spread), eval_floor(A, g["u"]))
    assert np.all(np.abs(got - want) <= tol), (got - want) / want
    s_got = np.array([h.s_hat for h in hist[1:]])
    assert np.array_equal(s_got == 0.0, g["hist"][1:, 5] == 0.0)
    scale = np.max(np.abs(g["u"]))
    assert np.max(np.abs(u - g["u"])) <= 1e-10 * scale
    if exact is not None:
        assert abs(hist[-1].err_max - g["hist"][-1, 3]) <= 1e-10 * max(1.0, g["hist"][-1, 3]) + 1e-13


def test_mt19937_64_known_answer():
    e = O.MT19937_64(5489)  # the standard's required 10000th output
    for _ in range(9999):
        e()
    assert e() == 9981545732273789042


def test_index_maps_partition():
    m = O.Mesh.create(2, [8, 8], [2, 2])
    holes = O.hole_positions(m)
    assert len(holes) == 36  # mesh.hpp example: 9 holes x 4 points
    skel = np.setdiff1d(np.arange(64), holes)
    assert len(skel) == 28
    for to in (1, 2, 3):
        mp = O.projector_map(m, 0, to)
        w = np.arange(1, len(mp) + 1, dtype=float)
        full = np.zeros(64)
        full[mp] = w
        assert np.array_equal(full[mp], w)  # gather-after-scatter identity (Prop. 2)
    with pytest.raises(O.DivisibilityError):
        O.Mesh.create(2, [10, 10], [4, 4])


def _fmt3(x):
    return float("%.3g" % x)


def test_reference_acceptance_figures_richardson_and_order():
    """test_output.txt criteria 10 and 11: ratio 3.99; extrapolated 0.00063 vs 0.0138, 0.0138, 0.0272."""
    p = O.reference_example(1, 1)
    m = O.Mesh.create(2, [24, 24], [4, 4])

    def direct(mask):
        A = O.assemble_operator(m, p, mask)
        return O.spla.splu(A.tocsc()).solve(O.assemble_rhs(m, p, mask))

    u1 = direct(2)[O.projector_map(m, 2, 3)]
    u2 = direct(1)[O.projector_map(m, 1, 3)]
    ucc = direct(3)
    uh = u1 + u2 - ucc
    x = O.coords(m, 3)[0]
    ex = p.exact(x)
    errs = [np.max(np.abs(v - ex)) for v in (uh, u1, u2, ucc)]
    assert [_fmt3(e) for e in errs] == [0.00063, 0.0138, 0.0138, 0.0272]

    def fine_err(nf):
        mm = O.Mesh.create(2, [nf, nf], [4, 4])
        A = O.assemble_operator(mm, p, 0)
        u = O.spla.splu(A.tocsc()).solve(O.assemble_rhs(mm, p, 0))
        return np.max(np.abs(u - p.exact(O.coords(mm, 0)[0])))

    assert _fmt3(fine_err(24) / fine_err(49)) == 3.99


def test_reference_acceptance_figures_initial_gap():
    """test_output.txt criterion 8: r0 = 24.9 vs 2.16e+04 (example 1, settings 1/2, 99/4)."""
    m = O.Mesh.create(2, [99, 99], [4, 4])
    r0 = []
    for setting in (1, 2):
        p = O.reference_example(1, setting)
        ctx = O.SolverContext(m, p)
        u = ctx.initial_guess(ctx.assembled_bundle(), O.mix_seed(0, 0), normalize=False)
        r0.append(float(np.linalg.norm(O.residual(ctx.A, ctx.b, u))))
    assert [_fmt3(x) for x in r0] == [24.9, 21600.0]


def test_reference_acceptance_figures_trend():
    """test_output.txt criterion 7: r1/r0 = 0.322, step ratio 0.998, stall 0.044 (nc=9) vs 0.00378 (nc=19)."""
    p = O.reference_example(1, 1)
    m9 = O.Mesh.create(2, [399, 399], [9, 9])
    _, _, h9, _ = O.asdsm_iterate(m9, p, 20, 0)
    m19 = O.Mesh.create(2, [399, 399], [19, 19])
    _, _, h19, _ = O.asdsm_iterate(m19, p, 20, 0)
    assert _fmt3(h9[1].res_l2 / h9[0].res_l2) == 0.322
    assert _fmt3(h9[20].res_l2 / h9[19].res_l2) == 0.998
    assert _fmt3(h9[-1].res_l2) == 0.044
    assert _fmt3(h19[-1].res_l2) == 0.00378


def test_reference_acceptance_figures_cross_residual():
    """test_output.txt criterion 9: max |r| = 0.000184 at distance 5 (steady toy), 0.00148 at
    distance 1 (space-time toy) after 20 iterations at 99/9."""
    out = []
    for ex, st in ((2, 1), (2, 2)):
        p = O.reference_example(ex, st)
        m = O.Mesh.create(2, [99, 99], [9, 9], 1 if p.time_dependent else -1)
        _, r, _, _ = O.asdsm_iterate(m, p, 20, 0)
        k = int(np.argmax(np.abs(r)))
        idx = (k % 99 + 1, k // 99 + 1)
        dist = 0
        for a in range(2):
            near = int(round(idx[a] / m.n[a])) * m.n[a]
            near = min(max(near, 0), (m.nc[a] + 1) * m.n[a])
            dist = max(dist, abs(idx[a] - near))
        out.append((_fmt3(float(np.max(np.abs(r)))), dist))
    assert out == [(0.000184, 5), (0.00148, 1)]
