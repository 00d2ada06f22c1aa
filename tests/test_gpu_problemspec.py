"""GPU tests of the caller-defined ProblemSpec boundary (C-ABI asdsm_problem_create) and of the
IterateOptions::observer counterpart (asdsm_iterate_observed).

The ProblemSpec fields restate the reference's example 1 (problems.cpp:13-43) as Python
callables; the plan samples them at the reference's assembly points, so the solve must be
bitwise the catalogue problem's (same operator, same right-hand sides, same path): the
constant-coefficient fields take the separable solvers, the variable ones the per-point path.
"""
import math

import numpy as np
import pytest

import paper_2303_01163_b200 as pb

pytestmark = pytest.mark.gpu
PI = math.pi


def ex1_setting1():  # problems.cpp:13-25
    exact = lambda x: math.sin(PI * x[0] + PI * x[1])  # noqa: E731

    def source(x):
        th = PI * x[0] + PI * x[1]
        return 2.0 * PI * PI * math.sin(th) + 2.0 * PI * math.cos(th)
    one = lambda x: 1.0  # noqa: E731
    return pb.ProblemSpec(2, [one, one], [one, one], source, exact, exact)


def ex1_setting2():  # problems.cpp:27-43
    exact = lambda x: math.sin(4.0 * PI * x[0] + 4.0 * PI * x[1])  # noqa: E731

    def source(x):
        th = 4.0 * PI * (x[0] + x[1])
        a = 3.0 + x[0] * x[0] + x[0] * x[1]
        b = 3.0 - x[0] + x[1]
        return 16.0 * PI * PI * a * math.sin(th) + 4.0 * PI * b * math.cos(th)
    return pb.ProblemSpec(2, [lambda x: 1.0 + x[0] * x[0], lambda x: 2.0 + x[0] * x[1]],
                          [lambda x: 2.0 - x[0], lambda x: 1.0 + x[1]], source, exact, exact)


def _hist(st):
    return np.array([[h.res_l2, h.res_inf, h.err_max, h.err_l2] for h in st.history])


@pytest.mark.parametrize("spec,setting,variable", [(ex1_setting1, 1, False), (ex1_setting2, 2, True)])
def test_problem_spec_matches_catalogue(spec, setting, variable):
    mesh = pb.asdsm.example_mesh(1, setting, 49, 4)
    opts = pb.IterateOptions(tol=0.0, max_iter=6, stagnation_window=0, rng_seed=2)
    ctx = pb.SolverContext(mesh, spec().problem())
    assert ctx.variable() == variable
    st = ctx.iterate(opts)
    ref = pb.SolverContext(mesh, pb.make_problem(1, setting)).iterate(opts)
    assert np.array_equal(_hist(st), _hist(ref))
    assert np.array_equal(st.u, ref.u)


def test_problem_spec_rejects_bad_fields():
    bad = pb.ProblemSpec(2, [lambda x: 1.0, lambda x: -1.0], [lambda x: 0.0, lambda x: 0.0], lambda x: 1.0,
                         lambda x: 0.0)
    with pytest.raises(pb.Error):
        pb.SolverContext(pb.MeshConfig.create(2, [19, 19], [4, 4]), bad.problem())


def test_observer_sees_every_record():
    """observer (solver.hpp:65): called after each record, k = 0 first, with the state at that
    point -- here checked against separate solves stopped at max_iter = k (bitwise: the observed
    run and the graph run do the same arithmetic)."""
    mesh = pb.asdsm.example_mesh(1, 1, 99, 9)
    seen = []
    opts = pb.IterateOptions(tol=0.0, max_iter=5, stagnation_window=0, rng_seed=1,
                             observer=lambda st: seen.append((len(st.history), st.u, st.history[-1].res_l2)))
    ctx = pb.SolverContext(mesh, pb.make_problem(1, 1))
    final = ctx.iterate(opts)
    assert [s[0] for s in seen] == list(range(1, 7))
    plain = ctx.iterate(pb.IterateOptions(tol=0.0, max_iter=5, stagnation_window=0, rng_seed=1))
    assert np.array_equal(_hist(final), _hist(plain)) and np.array_equal(final.u, plain.u)
    for k in (0, 2, 5):
        st = ctx.iterate(pb.IterateOptions(tol=0.0, max_iter=k, stagnation_window=0, rng_seed=1))
        assert np.array_equal(seen[k][1], st.u)
        assert seen[k][2] == st.history[-1].res_l2


def _advective(eps):
    one = lambda x: 1.0  # noqa: E731
    return pb.ProblemSpec(2, [lambda x: eps, lambda x: eps], [one, lambda x: 0.5],
                          lambda x: math.exp(-((x[0] - 0.3) ** 2 + (x[1] - 0.4) ** 2) / 0.02), lambda x: 0.0)


def test_strong_advection_falls_back_to_block_thomas(monkeypatch):
    """Constant coefficients the separable solvers cannot take (cell Peclet 5 on 49-point holes:
    no stable eigenvector scaling on either axis) run on the block-Thomas path with the same
    operator instead of raising Unsupported; the switch is visible as a variable plan."""
    mesh = pb.MeshConfig.create(2, [199, 199], [3, 3])
    opts = pb.IterateOptions(tol=0.0, max_iter=4, stagnation_window=0, rng_seed=5)
    ctx = pb.SolverContext(mesh, _advective(1e-3).problem())
    assert ctx.variable()
    st = ctx.iterate(opts)
    assert np.all(np.isfinite(st.u)) and st.history[-1].res_l2 < st.history[0].res_l2
    ok = pb.SolverContext(mesh, _advective(1e-1).problem())  # mild advection: separable solvers
    assert not ok.variable()
    monkeypatch.setenv("ASDSM_NO_SEPARABLE_FALLBACK", "1")
    with pytest.raises(pb.Unsupported):
        pb.SolverContext(mesh, _advective(1e-3).problem())
