"""GPU parity: the CUDA path (through the C-ABI) against the compiled reference oracle.

Tolerances:
  * index maps, residual evaluation: bit-exact.
  * initial guess / final solution: max-norm relative 1e-10.
  * per-iteration residual norms: |d res_k| <= res_k * max(1e-10, 10 * spread_k), where
    spread_k is the reference's own reproducibility floor up to iteration k (relative spread of
    its history when re-run with a different, equally valid fill ordering of its direct solver:
    Cuthill-McKee instead of reverse Cuthill-McKee; ref_tools.history_tolerance).
"""
import numpy as np
import pytest

import paper_2303_01163_b200 as pb
from ref_tools import (csr_residual_exact, have_ref, history_tolerance, ref_bundle, ref_error_guess, ref_iterate,
                       ref_iterate_pair, ref_maps)

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")]


def _ctx(spec, nf, nc):
    if spec.startswith("ex:"):
        _, e, s = spec.split(":")
        prob = pb.make_problem(int(e), int(s))
        mesh = pb.asdsm.example_mesh(int(e), int(s), nf, nc)
    else:
        _, cid, seed = spec.split(":")
        prob = pb.baseline_problem(int(cid), int(seed))
        mesh, _ = pb.baseline_mesh(int(cid))
        if nf:
            mesh = pb.MeshConfig.create(mesh.dim, [nf] * mesh.dim, [nc] * mesh.dim, mesh.time_axis)
    return pb.SolverContext(mesh, prob), mesh, prob


@pytest.mark.parametrize("spec,nf,nc", [("ex:1:1", 24, 4), ("ex:4:1", 14, 4), ("cfg:4:3", 29, 4), ("ex:3:1", 19, 4)])
def test_index_maps_bit_exact(spec, nf, nc):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    ref = ref_maps(spec, nf, nc)
    for key, m in ref.items():
        if key == "holes":
            continue
        fr, to = key
        got = ctx.projector_map(pb.MeshKind.from_mask(mesh.dim, fr), pb.MeshKind.from_mask(mesh.dim, to))
        assert np.array_equal(got, m), (fr, to)
    got = pb.hole_positions(mesh, ctx)
    assert np.array_equal(got, ref["holes"])


@pytest.mark.parametrize("spec,nf,nc", [("ex:1:1", 99, 9), ("cfg:2:5", 199, 9), ("ex:3:1", 49, 4),
                                        ("ex:4:1", 24, 4), ("cfg:4:1", 29, 4)])
def test_residual_bit_exact(spec, nf, nc):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    bun = ref_bundle(spec, nf, nc)
    assert np.array_equal(ctx.bundle["fine"], bun["fine"])  # host assembly == reference assembly
    for a in range(mesh.dim):
        assert np.array_equal(ctx.bundle["aniso"][a], bun["aniso"][a])
    assert np.array_equal(ctx.bundle["coarse"], bun["coarse"])
    rng = np.random.default_rng(7)
    u = rng.standard_normal(ctx.fine_size())
    r = ctx.residual(u)
    want = csr_residual_exact(bun, u)
    assert np.array_equal(r, want)


@pytest.mark.parametrize("spec,nf,nc", [("ex:1:1", 99, 9), ("cfg:0:0", 0, 0), ("cfg:1:2", 199, 9),
                                        ("cfg:2:5", 199, 9), ("ex:3:1", 99, 9)])
def test_initial_guess(spec, nf, nc):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    ref = ref_iterate(spec, nf, nc, 0, 0)
    u0 = ctx.initial_guess()
    scale = np.max(np.abs(ref["u0"]))
    assert np.max(np.abs(u0 - ref["u0"])) <= 1e-10 * scale


@pytest.mark.parametrize("spec,nf,nc,seed", [("ex:1:1", 99, 9, 3), ("cfg:2:5", 199, 9, 11)])
def test_error_guess_and_scaling(spec, nf, nc, seed):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    ref = ref_iterate(spec, nf, nc, 0, 0)
    r0 = ref["r0"]
    e_ref, s_ref = ref_error_guess(spec, nf, nc, seed, r0)
    e = ctx.error_guess(r0, seed)
    assert np.max(np.abs(e - e_ref)) <= 1e-10 * np.max(np.abs(e_ref))
    s = ctx.optimal_scaling(r0, e)
    assert abs(s - s_ref) <= 1e-10 * abs(s_ref)


def check_history(st, ref, alts):
    """GPU history and final iterate against the reference run `ref` (alts: the same run under
    other fill orderings, for the reproducibility floor)."""
    got = np.array([h.res_l2 for h in st.history])
    want = ref["hist"][:, 1]
    assert len(got) == len(want)
    tol = history_tolerance(ref, alts)
    bad = np.abs(got - want) > tol
    assert not bad.any(), list(zip(np.nonzero(bad)[0], got[bad], want[bad], tol[bad]))
    s_got = np.array([h.s_hat for h in st.history[1:]])
    assert np.array_equal(s_got == 0.0, ref["hist"][1:, 5] == 0.0)  # same accept/revert decisions
    scale = np.max(np.abs(ref["u"]))
    assert np.max(np.abs(st.u - ref["u"])) <= 1e-10 * scale
    return float(np.max(np.abs(got - want) / want)), float(np.max(np.abs(st.u - ref["u"])) / scale)


def assert_variant_ran(ctx_a, ctx_b):
    """Two plans of an A/B test really launched different kernels (the switch took effect)."""
    ka, kb = ctx_a.kernels(), ctx_b.kernels()
    assert ka and kb and set(ka) != set(kb), (sorted(ka), sorted(kb))


@pytest.mark.parametrize("spec,nf,nc,iters,seed", [
    ("cfg:0:0", 0, 0, 10, 0),
    ("ex:1:1", 99, 9, 20, 0),
    ("ex:3:1", 99, 9, 20, 0),
    ("cfg:1:2", 199, 9, 20, 1),
    ("cfg:2:5", 199, 9, 20, 2),
    ("cfg:1:0", 0, 0, 20, 0),  # the headline mesh at full size (one-launch slab step path)
    ("ex:1:1", 459, 3, 10, 2),  # holes of 114 x 114: the two-launch hole path (ring + partitioned lines)
])
def test_iterate_history(spec, nf, nc, iters, seed):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    ref, alts = ref_iterate_pair(spec, nf, nc, iters, seed)
    st = ctx.iterate(pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=seed))
    check_history(st, ref, alts)


@pytest.mark.parametrize("spec,nf,nc", [("ex:4:1", 24, 4), ("cfg:3:0", 29, 4), ("cfg:4:3", 29, 4)])
def test_initial_guess_3d(spec, nf, nc):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    ref = ref_iterate(spec, nf, nc, 0, 0)
    u0 = ctx.initial_guess()
    scale = np.max(np.abs(ref["u0"]))
    assert np.max(np.abs(u0 - ref["u0"])) <= 1e-10 * scale


@pytest.mark.parametrize("spec,nf,nc,iters,seed", [
    ("ex:4:1", 24, 4, 10, 0),
    ("cfg:3:0", 29, 4, 10, 1),
    ("cfg:4:3", 29, 4, 10, 2),
    ("cfg:3:0", 39, 9, 6, 0),
])
def test_iterate_history_3d(spec, nf, nc, iters, seed):
    test_iterate_history(spec, nf, nc, iters, seed)


@pytest.mark.parametrize("spec,nf,nc,iters", [("ex:1:2", 24, 4, 10), ("ex:1:2", 99, 9, 20), ("ex:3:2", 99, 9, 20),
                                              ("ex:4:2", 24, 4, 5)])
def test_variable_coefficients_match_reference(spec, nf, nc, iters):
    """Reference examples with variable alpha/beta (setting 2): per-point stencils and
    block-Thomas direct solves on the device."""
    ctx, mesh, prob = _ctx(spec, nf, nc)
    assert not prob.constant_coeffs and ctx.variable()
    bun = ref_bundle(spec, nf, nc)
    rng = np.random.default_rng(3)
    u = rng.standard_normal(ctx.fine_size())
    assert np.array_equal(ctx.residual(u), csr_residual_exact(bun, u))  # per-point stencil, bitwise
    ref, alts = ref_iterate_pair(spec, nf, nc, iters, 0)
    st = ctx.iterate(pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=0))
    check_history(st, ref, alts)


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:1:0", 0, 0, 20), ("cfg:1:2", 999, 9, 10)])
def test_slab_step_kernels_agree(spec, nf, nc, iters, monkeypatch):
    """The one-launch 2D slab step (slabstep2d.cu: partitioned warp line solves, DSMEM cross
    values, reciprocal-multiply normalization) against the three-launch path (PCR slab solves,
    last-block cc/spline, skeleton write): same iteration to rounding, on the headline mesh
    class.  Both are also checked against the reference by test_iterate_history."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=3)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_new = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_NO_SLABSTEP", "1")
    ctx_old, _, _ = _ctx(spec, nf, nc)
    st_old = ctx_old.iterate(opts)
    assert_variant_ran(ctx, ctx_old)
    a = np.array([h.res_l2 for h in st_new.history])
    b = np.array([h.res_l2 for h in st_old.history])
    assert len(a) == len(b)
    # the two paths round differently (reciprocal multiplies, partitioned vs cyclic-reduction
    # line solves); the fixed-point iteration carries those last-bit differences forward, so
    # the bound grows with k like the reference's own reordering spread does
    k = np.arange(len(b))
    assert np.all(np.abs(a - b) <= b * 1e-11 * 10.0 ** (k / 4.0) + 1e-14 * b[0])
    assert np.max(np.abs(st_new.u - st_old.u)) <= 1e-8 * np.max(np.abs(st_old.u))


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 6), ("cfg:4:1", 99, 4, 5), ("ex:1:1", 399, 4, 10)])
def test_even_odd_transforms_agree(spec, nf, nc, iters, monkeypatch):
    """The even/odd-split DMMA transforms (half sine table, dmma_gemm.cu) against the dense
    eigenvector GEMMs on meshes with axes of 64+ modes (the reference-parity tests above run
    coarser meshes).  The two round differently and the iteration amplifies last-bit
    differences (3D: ~1e-12 at k = 0 growing to ~1e-9), so the bound only has to catch a wrong
    transform, which would be off at O(1)."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=1)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_eo = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_DENSE_GEMM", "1")
    ctx_d, _, _ = _ctx(spec, nf, nc)
    st_d = ctx_d.iterate(opts)
    assert_variant_ran(ctx, ctx_d)
    a = np.array([h.res_l2 for h in st_eo.history])
    b = np.array([h.res_l2 for h in st_d.history])
    assert len(a) == len(b)
    assert np.all(np.abs(a - b) <= 1e-6 * b)
    assert np.max(np.abs(st_eo.u - st_d.u)) <= 1e-6 * np.max(np.abs(st_d.u))


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 6), ("cfg:3:0", 79, 4, 4),
                                              ("cfg:4:1", 99, 4, 5), ("cfg:4:1", 254, 4, 3),
                                              # m = 63 / 35: CAUSAL line ownership with 8 / 3 lines per
                                              # thread (the 8-slot kernel; config 4's m = 50 takes 5)
                                              ("cfg:4:1", 127, 1, 2), ("cfg:4:1", 71, 1, 2)])
def test_fused_hole3d_fill_agrees(spec, nf, nc, iters, monkeypatch):
    """The one-kernel 3D hole fill (holes3d_fused.cu: faces, line solves and both DMMA back
    transforms per hole in shared memory; SYM schedule for the steady configs, CAUSAL plane
    streaming for the space-time ones, m = 15 ... 50) against the four-launch path (faces kernel,
    Thomas kernel, two dense transform GEMMs).  One error guess must agree to rounding; the
    iteration amplifies last-bit differences, so its bound only has to catch a wrong fill."""
    ctx, _, _ = _ctx(spec, nf, nc)
    rng = np.random.default_rng(5)
    r = rng.standard_normal(ctx.fine_size())
    e_new = ctx.error_guess(r, 7)
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=1)
    st_new = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_HOLE3D_UNFUSED", "1")
    ctx_o, _, _ = _ctx(spec, nf, nc)
    e_old = ctx_o.error_guess(r, 7)
    st_old = ctx_o.iterate(opts)
    assert_variant_ran(ctx, ctx_o)
    assert np.max(np.abs(e_new - e_old)) <= 1e-12 * np.max(np.abs(e_old))
    a = np.array([h.res_l2 for h in st_new.history])
    b = np.array([h.res_l2 for h in st_old.history])
    assert len(a) == len(b)
    assert np.all(np.abs(a - b) <= 1e-6 * b)
    assert np.max(np.abs(st_new.u - st_old.u)) <= 1e-6 * np.max(np.abs(st_old.u))


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 5), ("cfg:4:1", 99, 4, 5), ("cfg:3:0", 29, 4, 6)])
def test_partitioned_slab_lines_agree(spec, nf, nc, iters, monkeypatch):
    """Slab line solves by the warp partition method (sepsolve.cu part_line_kernel: segment
    Thomas in registers + shuffle PCR over the separators) against the cyclic-reduction CTA per
    line (pcr_kernel).  Both are exact tridiagonal solvers; one error guess agrees to rounding."""
    ctx, _, _ = _ctx(spec, nf, nc)
    rng = np.random.default_rng(11)
    r = rng.standard_normal(ctx.fine_size())
    e_new = ctx.error_guess(r, 3)
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=2)
    st_new = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_PCR_LINES", "1")
    ctx_o, _, _ = _ctx(spec, nf, nc)
    e_old = ctx_o.error_guess(r, 3)
    st_old = ctx_o.iterate(opts)
    assert_variant_ran(ctx, ctx_o)
    assert np.max(np.abs(e_new - e_old)) <= 1e-11 * np.max(np.abs(e_old))
    a = np.array([h.res_l2 for h in st_new.history])
    b = np.array([h.res_l2 for h in st_old.history])
    assert np.all(np.abs(a - b) <= 1e-6 * b)


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 5), ("cfg:4:1", 99, 9, 4), ("ex:1:1", 399, 9, 6)])
def test_small_axis_transform_agrees(spec, nf, nc, iters, monkeypatch):
    """Short-axis eigenvector transforms as a thread-per-line stream (sepsolve.cu
    small_transform_kernel, m <= 16: the coarse axis of every slab) against the tiled DMMA GEMM."""
    ctx, _, _ = _ctx(spec, nf, nc)
    rng = np.random.default_rng(13)
    r = rng.standard_normal(ctx.fine_size())
    e_new = ctx.error_guess(r, 5)
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=6)
    st_new = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_NO_SMALL_TRANSFORM", "1")
    ctx_o, _, _ = _ctx(spec, nf, nc)
    e_old = ctx_o.error_guess(r, 5)
    st_old = ctx_o.iterate(opts)
    assert_variant_ran(ctx, ctx_o)
    assert np.max(np.abs(e_new - e_old)) <= 1e-11 * np.max(np.abs(e_old))
    a = np.array([h.res_l2 for h in st_new.history])
    b = np.array([h.res_l2 for h in st_old.history])
    assert np.all(np.abs(a - b) <= 1e-6 * b)


@pytest.mark.parametrize("spec,nf,nc", [("cfg:3:0", 129, 4), ("cfg:4:1", 99, 4), ("cfg:2:5", 0, 0), ("ex:4:1", 24, 4)])
def test_hole_rhs_rows_bitwise(spec, nf, nc, monkeypatch):
    """The row-per-CTA smooth-mode hole right-hand side (kernels.cu hole_rhs_rows_kernel) is the
    same arithmetic as the generic kernel: the initial guesses agree bitwise."""
    ctx, _, _ = _ctx(spec, nf, nc)
    u_new = ctx.initial_guess()
    monkeypatch.setenv("ASDSM_HOLE_RHS_OLD", "1")
    ctx_o, _, _ = _ctx(spec, nf, nc)
    u_old = ctx_o.initial_guess()
    assert np.array_equal(u_new, u_old)


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:1:0", 0, 0, 6), ("cfg:0:0", 0, 0, 10), ("cfg:3:0", 29, 4, 4)])
def test_one_call_solve(spec, nf, nc, iters):
    """asdsm_solve (uploads + solve + one-sync fetch) against set_bundle + asdsm_iterate: bitwise.
    With b scaled by 2 every stage is exactly homogeneous (zero initial guess, power-of-two
    scaling through the normalizations, value-independent cross-point draws), so u, r and the
    step s_hat double bit for bit."""
    ctx, mesh, _ = _ctx(spec, nf, nc)
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=3)
    st0 = ctx.iterate(opts)
    bun = {k: ([2.0 * x for x in v] if k == "aniso" else 2.0 * v) for k, v in ctx.bundle.items()}
    base = ctx.bundle
    st2 = ctx.solve(bun, None, opts)
    assert np.array_equal(st2.u, 2.0 * st0.u) and np.array_equal(st2.r, 2.0 * st0.r)
    # s_hat scales with b too: the error-mode correction is normalized
    assert np.array_equal([h.s_hat for h in st2.history], [2.0 * h.s_hat for h in st0.history], equal_nan=True)
    st1 = ctx.solve(base, None, opts)
    assert np.array_equal(st1.u, st0.u) and np.array_equal(st1.r, st0.r)
    assert [h.res_l2 for h in st1.history] == [h.res_l2 for h in st0.history]
    assert st1.stop_reason == st0.stop_reason


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:1:0", 0, 0, 20), ("ex:3:1", 199, 9, 12)])
def test_dots_update_launch_agrees(spec, nf, nc, iters, monkeypatch):
    """The opt-in single launch of the step dots and the update (ASDSM_DOTS_UPDATE=1: grid
    barrier on DevState::gen, cooperative launch) against the two-launch default: the dot
    products are summed over a different block split, so the step differs in the last bits."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=5)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_two = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_DOTS_UPDATE", "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_one = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    a = np.array([h.res_l2 for h in st_one.history])
    b = np.array([h.res_l2 for h in st_two.history])
    k = np.arange(len(b))
    assert len(a) == len(b)
    assert np.all(np.abs(a - b) <= b * 1e-11 * 10.0 ** (k / 4.0) + 1e-14 * b[0])
    assert np.max(np.abs(st_one.u - st_two.u)) <= 1e-8 * np.max(np.abs(st_two.u))


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 5), ("cfg:4:1", 99, 9, 4), ("ex:4:1", 24, 4, 6)])
def test_skel3d_dots_rows_agree(spec, nf, nc, iters, monkeypatch):
    """3D skeleton-plane step dots, one warp per skeleton row (default) against one thread per
    point (ASDSM_SKEL3D_POINTS=1): same points and per-point arithmetic, another summation order."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=2)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_rows = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_SKEL3D_POINTS", "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_pts = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    a = np.array([h.s_hat for h in st_rows.history[1:]])
    b = np.array([h.s_hat for h in st_pts.history[1:]])
    k = np.arange(1, len(b) + 1)
    # another summation order of the same dots: last-bit differences, amplified by the iteration
    assert np.all(np.abs(a - b) <= np.abs(b) * 1e-12 * 10.0 ** (k / 2.0) + 1e-300)
    assert np.max(np.abs(st_rows.u - st_pts.u)) <= 1e-10 * np.max(np.abs(st_pts.u))


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:2:5", 0, 0, 4), ("ex:1:1", 2049, 4, 4)])
def test_partitioned_hole_lines_agree(spec, nf, nc, iters, monkeypatch):
    """Large 2D holes (beyond the fused per-hole kernel): mode lines by one warp each with the
    partition method (default) against one thread each with Thomas (ASDSM_HOLE_THOMAS=1)."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=4)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_p = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_HOLE_THOMAS", "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_t = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    a = np.array([h.res_l2 for h in st_p.history])
    b = np.array([h.res_l2 for h in st_t.history])
    k = np.arange(len(b))
    assert len(a) == len(b)
    assert np.all(np.abs(a - b) <= b * 1e-11 * 10.0 ** (k / 4.0) + 1e-14 * b[0])
    assert np.max(np.abs(st_p.u - st_t.u)) <= 1e-8 * np.max(np.abs(st_t.u))


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 5), ("cfg:4:1", 99, 9, 4), ("ex:4:1", 24, 4, 6)])
def test_merge3d_warp_splines_bitwise(spec, nf, nc, iters, monkeypatch):
    """3D merge splines one warp per line (default) against one thread per line
    (ASDSM_M3_THREAD_LINES=1): the same operations in the same order, so bitwise the same solve."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=6)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_w = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_M3_THREAD_LINES", "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_t = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    assert np.array_equal(st_w.u, st_t.u) and np.array_equal(st_w.r, st_t.r)


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 5), ("cfg:4:1", 99, 9, 4), ("ex:4:1", 24, 4, 6)])
def test_stream3d_tma_pass_bitwise(spec, nf, nc, iters, monkeypatch):
    """The opt-in TMA-staged 3D update / residual pass (ASDSM_STREAM3D=1, stream3d.cu: pair-row
    tensor maps, v = u + s e formed once per point) against the default axpy + z-coarsened
    residual passes: the same row sums in the reference's CSR order, so bitwise the same solve."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=3)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_d = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_STREAM3D", "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_t = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    assert any("stream3d_kernel" in k for k in ctx1.kernels()), sorted(ctx1.kernels())
    assert np.array_equal(st_d.u, st_t.u) and np.array_equal(st_d.r, st_t.r)
    # (the norms are reduced over another grid shape: the same values summed in another order)
    a = np.array([h.res_l2 for h in st_d.history])
    b = np.array([h.res_l2 for h in st_t.history])
    assert np.all(np.abs(a - b) <= 1e-14 * b)


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:0:0", 0, 0, 6), ("cfg:1:2", 199, 9, 6), ("cfg:2:5", 199, 9, 6),
                                              ("cfg:1:0", 0, 0, 5), ("ex:1:1", 459, 3, 4)])
def test_ymarch2d_pass_bitwise(spec, nf, nc, iters, monkeypatch):
    """The lean y-march of the 2D residual / update pass (default, march.cu stencil2d_ym_kernel:
    clamped neighbour offsets with zeroed edge coefficients, station copies from a uniform row
    test) against the tile-walking kernel with per-point boundary predicates (ASDSM_YC2D=1): the
    same row sums in the reference's CSR order (fdm.cpp:110-117), so bitwise the same solve."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=3)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_d = ctx.iterate(opts)
    assert any("stencil2d_ym_kernel" in k for k in ctx.kernels()), sorted(ctx.kernels())
    monkeypatch.setenv("ASDSM_YC2D", "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_t = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    assert np.array_equal(st_d.u, st_t.u) and np.array_equal(st_d.r, st_t.r)
    a = np.array([h.res_l2 for h in st_d.history])
    b = np.array([h.res_l2 for h in st_t.history])
    assert np.all(np.abs(a - b) <= 1e-14 * b)


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:2:5", 0, 0, 4), ("ex:1:1", 2049, 4, 4)])
def test_strip_back_resident_agrees(spec, nf, nc, iters, monkeypatch):
    """Strip back transform with the half sine table resident in shared memory (default,
    dmma_gemm.cu strip_back_kernel: whole-K tiles, E and O in one thread) against the generic
    even/odd DMMA GEMM (ASDSM_STRIP_BACK=0): the same sums in the same k order."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=4)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_s = ctx.iterate(opts)
    assert any("strip_back_kernel" in k for k in ctx.kernels()), sorted(ctx.kernels())
    monkeypatch.setenv("ASDSM_STRIP_BACK", "0")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_w = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    a = np.array([h.res_l2 for h in st_s.history])
    b = np.array([h.res_l2 for h in st_w.history])
    k = np.arange(len(b))
    assert len(a) == len(b)
    assert np.all(np.abs(a - b) <= b * 1e-11 * 10.0 ** (k / 4.0) + 1e-14 * b[0])
    assert np.max(np.abs(st_s.u - st_w.u)) <= 1e-8 * np.max(np.abs(st_w.u))


@pytest.mark.parametrize("switch", ["ASDSM_ZC3D", "ASDSM_UPD3D_FUSED"])
@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:3:0", 129, 4, 5), ("cfg:4:1", 99, 9, 4), ("ex:4:1", 24, 4, 6)])
def test_zmarch3d_pass_bitwise(spec, nf, nc, iters, switch, monkeypatch):
    """The lean z-march of the 3D residual / candidate residual (default, march.cu
    stencil3d_zm_kernel: clamped neighbour offsets with zeroed edge coefficients) against the
    tile-walking z-coarsened kernel with per-point boundary predicates (ASDSM_ZC3D=1), and its
    fused update form (ASDSM_UPD3D_FUSED=1) against axpy + candidate residual: the same row sums
    in the reference's CSR order (fdm.cpp:110-117), so bitwise the same solve."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=3)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_d = ctx.iterate(opts)
    assert any("stencil3d_zm_kernel" in k for k in ctx.kernels()), sorted(ctx.kernels())
    monkeypatch.setenv(switch, "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_t = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    assert np.array_equal(st_d.u, st_t.u) and np.array_equal(st_d.r, st_t.r)
    # (the norms are reduced over another grid shape: the same values summed in another order)
    a = np.array([h.res_l2 for h in st_d.history])
    b = np.array([h.res_l2 for h in st_t.history])
    assert np.all(np.abs(a - b) <= 1e-14 * b)


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:2:5", 0, 0, 4), ("ex:1:1", 2049, 4, 4)])
def test_hole_strip_split_agrees(spec, nf, nc, iters, monkeypatch):
    """Large 2D holes split into strips (default: separator columns from the hole's own modes,
    then every strip solved as a hole with w-point transforms, holes2d.cu hole2d_sep_rows_kernel)
    against the whole-hole back transform (ASDSM_STRIPS=0): the same exact hole solve."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=4)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_s = ctx.iterate(opts)
    assert any("hole2d_sep_scatter_kernel" in k for k in ctx.kernels()), sorted(ctx.kernels())
    monkeypatch.setenv("ASDSM_STRIPS", "0")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_w = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    a = np.array([h.res_l2 for h in st_s.history])
    b = np.array([h.res_l2 for h in st_w.history])
    k = np.arange(len(b))
    assert len(a) == len(b)
    assert np.all(np.abs(a - b) <= b * 1e-11 * 10.0 ** (k / 4.0) + 1e-14 * b[0])
    assert np.max(np.abs(st_s.u - st_w.u)) <= 1e-8 * np.max(np.abs(st_w.u))


@pytest.mark.parametrize("spec,nf,nc,iters", [("cfg:2:5", 0, 0, 4), ("ex:1:1", 2049, 4, 4)])
def test_separator_gemm_agrees(spec, nf, nc, iters, monkeypatch):
    """The strip split's separators from one GEMM with the separator response matrix K (default;
    K built at plan creation from the iteration's own mode-line and separator kernels on unit
    rings) against the per-iteration mode lines + separator product (ASDSM_SEP_MODES=1)."""
    opts = pb.IterateOptions(tol=0.0, max_iter=iters, stagnation_window=0, rng_seed=4)
    ctx, _, _ = _ctx(spec, nf, nc)
    st_g = ctx.iterate(opts)
    monkeypatch.setenv("ASDSM_SEP_MODES", "1")
    ctx1, _, _ = _ctx(spec, nf, nc)
    st_m = ctx1.iterate(opts)
    assert_variant_ran(ctx, ctx1)
    assert any("hole2d_sep_rows_kernel" in k for k in ctx1.kernels()), sorted(ctx1.kernels())
    a = np.array([h.res_l2 for h in st_g.history])
    b = np.array([h.res_l2 for h in st_m.history])
    k = np.arange(len(b))
    assert np.all(np.abs(a - b) <= b * 1e-11 * 10.0 ** (k / 4.0) + 1e-14 * b[0])
    assert np.max(np.abs(st_g.u - st_m.u)) <= 1e-8 * np.max(np.abs(st_m.u))
