"""The reference's public solver stages (solver.hpp:70-105) through the C-ABI
(asdsm_richardson_extrapolate, asdsm_choose_cross_points, asdsm_spline_correct,
asdsm_build_skeleton, asdsm_merge_3d, asdsm_fill_holes) against the compiled reference
(oracle/_ref/ref_dump stage ...) on the same seeded random fields: the merge stages keep the
reference's operation order (solver.cpp:98-196, 297-410) -- bitwise; fill_holes solves the holes
directly -- within 1e-10 of the reference's sparse LU."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2303_01163_b200 as pb
from ref_tools import REF_DUMP, have_ref
from test_gpu_parity import _ctx

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")]


def _ref_stage(name, spec, nf, nc, seed, fields):
    with tempfile.TemporaryDirectory() as d:
        for k, v in fields.items():
            np.asarray(v, dtype=np.float64).tofile(os.path.join(d, f"in.{k}.f64"))
        subprocess.check_call([REF_DUMP, "stage", name, spec, str(nf), str(nc), str(seed), os.path.join(d, "in"),
                               os.path.join(d, "out")])
        return np.fromfile(os.path.join(d, "out.f64"))


def _kind(ctx, mask):
    return ctx.config.point_count(pb.MeshKind.from_mask(ctx.config.dim, mask))


def _hole_mask(mesh):
    nf, n = mesh.fine_counts, [f // c for f, c in zip([x + 1 for x in mesh.fine_counts], [x + 1 for x in mesh.coarse_counts])]
    idx = np.indices(tuple(reversed(nf))).reshape(mesh.dim, -1)[::-1]  # axis 0 fastest
    return np.all([(idx[a] + 1) % n[a] != 0 for a in range(mesh.dim)], axis=0)


@pytest.mark.parametrize("spec,nf,nc", [("ex:1:1", 49, 4), ("cfg:1:0", 99, 9)])
def test_stages_2d_match_reference(spec, nf, nc):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    rng = np.random.default_rng(7)
    ucc, u1, u2 = (rng.standard_normal(_kind(ctx, 3)) for _ in range(3))
    ufc, ucf = rng.standard_normal(_kind(ctx, 2)), rng.standard_normal(_kind(ctx, 1))
    got = ctx.richardson_extrapolate(u1, u2, ucc)
    assert np.array_equal(got, _ref_stage("richardson", spec, nf, nc, 0, {"u1": u1, "u2": u2, "ucc": ucc}))
    for seed in range(4):  # both seeded draws
        got = ctx.choose_cross_points(ufc, ucf, seed)
        assert np.array_equal(got, _ref_stage("choose", spec, nf, nc, seed, {"ufc": ufc, "ucf": ucf}))
    for dense, ua in ((0, ufc), (1, ucf)):
        got = ctx.spline_correct(ua, ucc, dense)
        assert np.array_equal(got, _ref_stage(f"spline{dense}", spec, nf, nc, 0, {"ua": ua, "ecc": ucc}))
    got = ctx.build_skeleton(ufc, ucf, ucc)
    want = _ref_stage("skeleton_s", spec, nf, nc, 0, {"ufc": ufc, "ucf": ucf, "ucc": ucc})
    assert np.array_equal(got, want), np.max(np.abs(got - want))
    for seed in (0, 1, 5):
        got = ctx.build_skeleton(ufc, ucf, None, normalized=True, rng_seed=seed)
        want = _ref_stage("skeleton_e", spec, nf, nc, seed, {"ufc": ufc, "ucf": ucf})
        assert np.array_equal(got, want), np.max(np.abs(got - want))
    with pytest.raises(pb.InvalidKind):
        ctx.build_skeleton(ufc, ucf, ucc, normalized=True)


@pytest.mark.parametrize("spec,nf,nc", [("ex:4:1", 24, 4), ("cfg:3:0", 29, 4)])
def test_merge_3d_matches_reference(spec, nf, nc):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    rng = np.random.default_rng(11)
    ux, uy, uz = (rng.standard_normal(_kind(ctx, 1 << a)) for a in range(3))
    uccc = rng.standard_normal(_kind(ctx, 7))
    got = ctx.merge_3d(ux, uy, uz, uccc)
    want = _ref_stage("merge_s", spec, nf, nc, 0, {"ux": ux, "uy": uy, "uz": uz, "uccc": uccc})
    assert np.array_equal(got, want), np.max(np.abs(got - want))
    for seed in (0, 3, 9):
        got = ctx.merge_3d(ux, uy, uz, None, seed)
        want = _ref_stage("merge_e", spec, nf, nc, seed, {"ux": ux, "uy": uy, "uz": uz})
        assert np.array_equal(got, want), np.max(np.abs(got - want))
    with pytest.raises(pb.InvalidKind):
        ctx.build_skeleton(np.zeros(_kind(ctx, 2)), np.zeros(_kind(ctx, 1)), None, normalized=True)


@pytest.mark.parametrize("spec,nf,nc", [("ex:1:1", 49, 4), ("cfg:2:1", 199, 9), ("ex:4:1", 24, 4), ("ex:1:2", 49, 4)])
def test_fill_holes_matches_reference(spec, nf, nc):
    ctx, mesh, _ = _ctx(spec, nf, nc)
    rng = np.random.default_rng(3)
    holes = _hole_mask(mesh)
    skel = np.where(holes, 0.0, rng.standard_normal(holes.size))
    b = rng.standard_normal(holes.size)
    for bb in (b, np.zeros_like(b)):
        got = ctx.fill_holes(skel, bb)
        want = _ref_stage("fill", spec, nf, nc, 0, {"skel": skel, "b": bb})
        assert np.array_equal(got[~holes], want[~holes])  # the skeleton passes through
        assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want)), np.max(np.abs(got - want))
    bad = skel.copy()
    bad[np.flatnonzero(holes)[3]] = 1.0
    with pytest.raises(pb.SkeletonNotHollow):
        ctx.fill_holes(bad, b)
