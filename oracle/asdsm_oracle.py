"""CPU restatement of the reference ASDSM algorithm (numpy/scipy).  TEST INFRASTRUCTURE ONLY.

This module is the oracle the parity tests check the B200 path against; nothing in the
product (paper_2303_01163_b200/) imports it.  Each function cites the reference file:line it
restates (reference: arxiv/paper_2303_01163, proj/).  Pinned against the reference itself:
tests/test_oracle_cpu.py compares it with golden vectors produced by the reference's own
sources compiled here (oracle/_ref, generator tests/golden/make_golden.py).

Direct solves use scipy's SuperLU (sparse LU with COLAMD and partial pivoting -- the same
published algorithm as the reference's Eigen::SparseLU<..., COLAMDOrdering<int>>,
proj/src/linsolve.cpp:28-66); rounding differs from Eigen's, see DESIGN.md "Parity".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

MASK64 = (1 << 64) - 1


# ------------------------------------------------------------------ seeds / RNG ------------
def mix_seed(base: int, k: int) -> int:
    """solver.cpp:88-96 (splitmix64 finalizer)."""
    z = (base + 0x9E3779B97F4A7C15 * (k + 1)) & MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


class MT19937_64:
    """std::mt19937_64 (the engine solver.cpp:118, 309 and 469 draw from)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64
        self.idx = 312

    def _twist(self):
        upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for i in range(312):
            x = (self.mt[i] & upper) | (self.mt[(i + 1) % 312] & lower)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            self.mt[i] = self.mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


# ------------------------------------------------------------------ mesh -------------------
class DivisibilityError(ValueError):
    pass


class DegenerateError(ValueError):
    pass


class ZeroNormSolution(ArithmeticError):
    pass


@dataclass
class Mesh:
    """MeshConfig (mesh.hpp:56-83), validation as MeshConfig::create (mesh.cpp:47-76)."""
    dim: int
    nf: List[int]
    nc: List[int]
    n: List[int]
    h: List[float]
    H: List[float]
    time_axis: int = -1

    @staticmethod
    def create(dim, nf, nc, time_axis=-1):
        n, h, H = [], [], []
        for a in range(dim):
            if nf[a] < 1 or nc[a] < 1:
                raise DegenerateError(f"axis {a}: interior point counts must be >= 1")
            if (nf[a] + 1) % (nc[a] + 1):
                raise DivisibilityError(f"axis {a}: fine intervals {nf[a] + 1} not divisible by coarse intervals {nc[a] + 1}")
            f = (nf[a] + 1) // (nc[a] + 1)
            if f < 2:
                raise DegenerateError(f"axis {a}: refinement factor 1 leaves no holes")
            n.append(f)
            h.append(1.0 / float(nf[a] + 1))
            H.append(float(f) * (1.0 / float(nf[a] + 1)))
        return Mesh(dim, list(nf), list(nc), n, h, H, time_axis)

    def ext(self, mask):
        return [self.nc[a] if (mask >> a) & 1 else self.nf[a] for a in range(self.dim)]

    def count(self, mask):
        return int(np.prod(self.ext(mask)))

    def fine_index(self, mask, a, t):
        """0-based fine index of kind-local 0-based index t on axis a."""
        return (t + 1) * self.n[a] - 1 if (mask >> a) & 1 else t


def multi_indices(ext):
    """0-based multi-indices of an x-fastest layout, as arrays per axis."""
    grids = np.meshgrid(*[np.arange(e) for e in ext], indexing="ij")
    return [g.reshape(-1, order="F") for g in grids]


def projector_map(mesh: Mesh, from_mask: int, to_mask: int) -> np.ndarray:
    """build_projector (mesh.cpp:210-256): target linear index -> source linear index."""
    if (from_mask & to_mask) != from_mask:
        raise ValueError("not a sub-mesh")
    t_ext, f_ext = mesh.ext(to_mask), mesh.ext(from_mask)
    idx = multi_indices(t_ext)
    src = np.zeros(len(idx[0]), dtype=np.int64)
    stride = 1
    for a in range(mesh.dim):
        step = mesh.n[a] if ((to_mask >> a) & 1) and not ((from_mask >> a) & 1) else 1
        src += ((idx[a] + 1) * step - 1) * stride
        stride *= f_ext[a]
    return src


def hole_positions(mesh: Mesh) -> np.ndarray:
    """Concatenated hole_blocks positions (mesh.cpp:258-305), block by block."""
    d = mesh.dim
    blocks = multi_indices([mesh.nc[a] + 1 for a in range(d)])
    inner = multi_indices([mesh.n[a] - 1 for a in range(d)])
    out = []
    for b in range(len(blocks[0])):
        lin = np.zeros(len(inner[0]), dtype=np.int64)
        stride = 1
        for a in range(d):
            lin += (blocks[a][b] * mesh.n[a] + inner[a]) * stride
            stride *= mesh.nf[a]
        out.append(lin)
    return np.concatenate(out)


def hole_blocks(mesh: Mesh):
    d = mesh.dim
    per = int(np.prod([mesh.n[a] - 1 for a in range(d)]))
    pos = hole_positions(mesh)
    return [pos[i * per:(i + 1) * per] for i in range(len(pos) // per)]


# ------------------------------------------------------------------ problems / fdm ---------
@dataclass
class Problem:
    """ProblemSpec (fdm.hpp:18-30): coefficient functions of x (array (3, npts))."""
    dim: int
    alpha: List[Callable]
    beta: List[Callable]
    source: Callable
    boundary: Callable
    exact: Optional[Callable] = None
    time_dependent: bool = False


def coords(mesh: Mesh, mask: int, origin=None, ext=None):
    ext = mesh.ext(mask) if ext is None else ext
    idx = multi_indices(ext)
    x = np.zeros((3, len(idx[0])))
    for a in range(mesh.dim):
        stride = mesh.n[a] if (mask >> a) & 1 else 1
        o = 0 if origin is None else origin[a]
        x[a] = (o + (idx[a] + 1) * stride).astype(np.float64) * mesh.h[a]
    return x, idx


def axis_coeffs(mesh: Mesh, prob: Problem, mask: int, x):
    """axis_coeffs (fdm.cpp:63-82) per axis: (left, right, diag part, has_right)."""
    out = []
    for a in range(mesh.dim):
        step = mesh.H[a] if (mask >> a) & 1 else mesh.h[a]
        if a == mesh.time_axis:
            tc = 1.0 / step
            out.append((np.full(x.shape[1], -tc), np.zeros(x.shape[1]), np.full(x.shape[1], tc), False))
            continue
        al = np.broadcast_to(prob.alpha[a](x), (x.shape[1],)).astype(np.float64)
        be = np.broadcast_to(prob.beta[a](x), (x.shape[1],)).astype(np.float64)
        c = al / (step * step)
        d = be / (2.0 * step)
        out.append((-c - d, -c + d, 2.0 * c, True))
    return out


def assemble_operator(mesh: Mesh, prob: Problem, mask: int, ext=None, origin=None):
    """assemble_core (fdm.cpp:84-126): CSR with columns in ascending order."""
    ext = mesh.ext(mask) if ext is None else ext
    x, idx = coords(mesh, mask, origin, ext)
    n = len(idx[0])
    co = axis_coeffs(mesh, prob, mask, x)
    diag = np.zeros(n)
    for a in range(mesh.dim):
        diag = diag + co[a][2]
    strides = np.cumprod([1] + list(ext[:-1]))
    rows, cols, vals = [], [], []
    lin = np.arange(n)
    for a in reversed(range(mesh.dim)):
        m = idx[a] > 0
        rows.append(lin[m]); cols.append(lin[m] - strides[a]); vals.append(co[a][0][m])
    rows.append(lin); cols.append(lin); vals.append(diag)
    for a in range(mesh.dim):
        if not co[a][3]:
            continue
        m = idx[a] < ext[a] - 1
        rows.append(lin[m]); cols.append(lin[m] + strides[a]); vals.append(co[a][1][m])
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    A.sort_indices()
    return A


def assemble_rhs(mesh: Mesh, prob: Problem, mask: int):
    """rhs_core (fdm.cpp:128-171): source plus Dirichlet lifting, same coordinates/order."""
    ext = mesh.ext(mask)
    x, idx = coords(mesh, mask)
    v = np.asarray(prob.source(x), dtype=np.float64).copy()
    co = axis_coeffs(mesh, prob, mask, x)
    for a in range(mesh.dim):
        stride = mesh.n[a] if (mask >> a) & 1 else 1
        m = idx[a] == 0
        if m.any():
            xb = x[:, m].copy()
            xb[a] = 0.0 * mesh.h[a]
            v[m] = v[m] - co[a][0][m] * prob.boundary(xb)
        m = idx[a] == ext[a] - 1
        if co[a][3] and m.any():
            xb = x[:, m].copy()
            xb[a] = float((ext[a] + 1) * stride) * mesh.h[a]
            v[m] = v[m] - co[a][1][m] * prob.boundary(xb)
    return v


def csr_matvec_ordered(A: sp.csr_matrix, u: np.ndarray) -> np.ndarray:
    """SparseMatrix::multiply (sparse.cpp:49-58): each row summed left to right from 0.0."""
    counts = np.diff(A.indptr)
    acc = np.zeros(A.shape[0])
    for slot in range(int(counts.max()) if len(counts) else 0):
        rows = np.nonzero(counts > slot)[0]
        k = A.indptr[rows] + slot
        acc[rows] = acc[rows] + A.data[k] * u[A.indices[k]]
    return acc


def residual(A, b, u):
    """residual (fdm.cpp:221-230)."""
    return b - csr_matvec_ordered(A, u)


# ------------------------------------------------------------------ spline -----------------
def zero_clamped_spline(knots, values):
    """zero_clamped_spline + CubicSpline ctor (spline.cpp:9-37, 58-76): second derivatives."""
    x = [0.0] + list(knots) + [1.0]
    y = [0.0] + list(values) + [0.0]
    n = len(x)
    m = [0.0] * n
    if n > 2:
        ni = n - 2
        diag, upper, rhs = [0.0] * ni, [0.0] * ni, [0.0] * ni
        for i in range(ni):
            hl = x[i + 1] - x[i]
            hr = x[i + 2] - x[i + 1]
            diag[i] = (hl + hr) / 3.0
            upper[i] = hr / 6.0
            rhs[i] = (y[i + 2] - y[i + 1]) / hr - (y[i + 1] - y[i]) / hl
        for i in range(1, ni):
            lower = (x[i + 1] - x[i]) / 6.0
            w = lower / diag[i - 1]
            diag[i] -= w * upper[i - 1]
            rhs[i] -= w * rhs[i - 1]
        m[ni] = rhs[ni - 1] / diag[ni - 1]
        for i in range(ni - 1, 0, -1):
            m[i] = (rhs[i - 1] - upper[i - 1] * m[i + 1]) / diag[i - 1]
    return np.array(x), np.array(y), np.array(m)


def spline_eval(spl, xs):
    """CubicSpline::operator() (spline.cpp:39-56), vectorized over xs."""
    x, y, m = spl
    n = len(x)
    i = np.searchsorted(x, xs, side="right")
    i = np.clip(i, 1, n - 1) - 1
    h = x[i + 1] - x[i]
    t = xs - x[i]
    c1 = (y[i + 1] - y[i]) / h - h * (2.0 * m[i] + m[i + 1]) / 6.0
    c2 = m[i] / 2.0
    c3 = (m[i + 1] - m[i]) / (6.0 * h)
    out = y[i] + t * (c1 + t * (c2 + t * c3))
    return np.where(xs == x[-1], y[-1], out)


def coarse_knots(mesh: Mesh, a: int):
    """coarse_knots (solver.cpp:36-42)."""
    return np.array([float(c * mesh.n[a]) * mesh.h[a] for c in range(1, mesh.nc[a] + 1)])


def fine_coords(mesh: Mesh, a: int):
    """fine_coords (solver.cpp:44-49)."""
    return np.array([float(i) * mesh.h[a] for i in range(1, mesh.nf[a] + 1)])


# ------------------------------------------------------------------ skeleton (2D) ----------
def _as_grid(mesh, mask, v):
    return v.reshape(tuple(reversed(mesh.ext(mask))))  # [.., y, x]


def build_skeleton_2d(mesh: Mesh, u_fc, u_cf, u_cc, coin_seed):
    """build_skeleton (solver.cpp:154-196) with richardson_extrapolate (98-108),
    choose_cross_points (110-120) and spline_correct (122-152)."""
    fc, cf, cc = 2, 1, 3  # coarse along y (dense x), coarse along x (dense y), both
    P_fc_cc = projector_map(mesh, fc, cc)
    P_cf_cc = projector_map(mesh, cf, cc)
    u1 = u_fc[P_fc_cc]
    u2 = u_cf[P_cf_cc]
    if u_cc is not None:
        uh = u1 + u2 - u_cc
    else:
        eng = MT19937_64(coin_seed)
        uh = u2.copy() if eng() % 2 == 0 else u1.copy()
    e1, e2 = uh - u1, uh - u2
    E1 = e1.reshape(mesh.nc[1], mesh.nc[0])  # [J, I]
    E2 = e2.reshape(mesh.nc[1], mesh.nc[0])
    ut_fc = _as_grid(mesh, fc, u_fc.copy())  # [J, i]
    kx, xs = coarse_knots(mesh, 0), fine_coords(mesh, 0)
    for J in range(mesh.nc[1]):
        ut_fc[J, :] = ut_fc[J, :] + spline_eval(zero_clamped_spline(kx, E1[J, :]), xs)
    ut_cf = _as_grid(mesh, cf, u_cf.copy())  # [j, I]
    ky, ys = coarse_knots(mesh, 1), fine_coords(mesh, 1)
    for I in range(mesh.nc[0]):
        ut_cf[:, I] = ut_cf[:, I] + spline_eval(zero_clamped_spline(ky, E2[:, I]), ys)
    out = np.zeros(mesh.count(0))
    np.add.at(out, projector_map(mesh, 0, fc), ut_fc.reshape(-1))
    np.add.at(out, projector_map(mesh, 0, cf), ut_cf.reshape(-1))
    np.add.at(out, projector_map(mesh, 0, cc), -ut_cf.reshape(-1)[P_cf_cc])
    return out


# ------------------------------------------------------------------ skeleton (3D) ----------
def merge_3d(mesh: Mesh, u, u_ccc, seed):
    """merge_3d (solver.cpp:297-410) with correct_slab_plane (200-293)."""
    nc, nf, n = mesh.nc, mesh.nf, mesh.n
    slab = [1, 2, 4]
    G = lambda mask, v: v.reshape(tuple(reversed(mesh.ext(mask)))).transpose(2, 1, 0)  # [x, y, z]
    U = [G(slab[a], u[a]) for a in range(3)]
    st = lambda a, c: (c + 1) * n[a] - 1
    ci = [np.arange(nc[a]) for a in range(3)]
    fi = [np.arange(nf[a]) for a in range(3)]
    S0 = U[0][np.ix_(ci[0], st(1, ci[1]), st(2, ci[2]))]
    S1 = U[1][np.ix_(st(0, ci[0]), ci[1], st(2, ci[2]))]
    S2 = U[2][np.ix_(st(0, ci[0]), st(1, ci[1]), ci[2])]
    S = [S0, S1, S2]
    eng = MT19937_64(seed)
    if u_ccc is not None:
        Uc = G(7, u_ccc)
        uh = (S[0] + S[1] + S[2] - Uc) / 2.0
    else:
        uh = S[eng() % 3].copy()
    T = {}
    for a in range(3):
        for b in range(a + 1, 3):
            f = 3 - a - b
            # projections of slab a and slab b onto the pair kind (coarse on a and b)
            def proj(src_axis, arr):
                sl = [None, None, None]
                for ax in range(3):
                    if ax == f:
                        sl[ax] = fi[f]
                    elif ax == src_axis:
                        sl[ax] = ci[ax]
                    else:
                        sl[ax] = st(ax, ci[ax])
                return arr[np.ix_(*sl)]
            ua_p, ub_p = proj(a, U[a]), proj(b, U[b])
            if u_ccc is not None:
                base = (ua_p + ub_p) / 2.0
                base_t = (S[a] + S[b]) / 2.0
            else:
                pick_b = eng() % 2 != 0
                base = (ub_p if pick_b else ua_p).copy()
                base_t = S[b] if pick_b else S[a]
            corr = uh - base_t
            knots, xs = coarse_knots(mesh, f), fine_coords(mesh, f)
            for Ca in range(nc[a]):
                for Cb in range(nc[b]):
                    sel = [None, None, None]
                    sel[a], sel[b] = Ca, Cb
                    sel[f] = slice(None)
                    vals = corr[tuple(sel)]
                    base[tuple(sel)] = base[tuple(sel)] + spline_eval(zero_clamped_spline(knots, vals), xs)
                    pin = list(sel)
                    pin[f] = st(f, ci[f])
                    base[tuple(pin)] = uh[tuple(sel)]
            T[(a, b)] = base
    corrected = [U[a].copy() for a in range(3)]
    for a in range(3):
        f1, f2 = (1 if a == 0 else 0), (1 if a == 2 else 2)
        T1, T2 = T[tuple(sorted((a, f1)))], T[tuple(sorted((a, f2)))]
        k1s, k2s = coarse_knots(mesh, f1), coarse_knots(mesh, f2)
        x1, x2 = fine_coords(mesh, f1), fine_coords(mesh, f2)
        for I in range(nc[a]):
            def plane(arr):  # arr indexed [x,y,z] -> 2D [f1, f2] at a=I
                sel = [slice(None)] * 3
                sel[a] = I
                return arr[tuple(sel)]
            Sp, T1p, T2p, Hp = plane(U[a]), plane(T1), plane(T2), plane(uh)
            d = np.zeros((nf[f1], nf[f2]))
            for k2 in range(nf[f2]):
                vals = T1p[:, k2] - Sp[st(f1, ci[f1]), k2]
                d[:, k2] = d[:, k2] + spline_eval(zero_clamped_spline(k1s, vals), x1)
            for k1 in range(nf[f1]):
                vals = T2p[k1, :] - Sp[k1, st(f2, ci[f2])]
                d[k1, :] = d[k1, :] + spline_eval(zero_clamped_spline(k2s, vals), x2)
            g = np.zeros((nf[f1], nc[f2]))
            for C2 in range(nc[f2]):
                vals = Hp[:, C2] - Sp[st(f1, ci[f1]), st(f2, C2)]
                g[:, C2] = spline_eval(zero_clamped_spline(k1s, vals), x1)
            for k1 in range(nf[f1]):
                d[k1, :] = d[k1, :] - spline_eval(zero_clamped_spline(k2s, g[k1, :]), x2)
            sel = [slice(None)] * 3
            sel[a] = I
            corrected[a][tuple(sel)] = corrected[a][tuple(sel)] + d
    out = np.zeros(mesh.count(0))
    F = lambda mask, arr: arr.transpose(2, 1, 0).reshape(-1)  # back to x-fastest
    for a in range(3):
        np.add.at(out, projector_map(mesh, 0, slab[a]), F(slab[a], corrected[a]))
    for a in range(3):
        for b in range(a + 1, 3):
            np.add.at(out, projector_map(mesh, 0, (1 << a) | (1 << b)), -F(0, T[(a, b)]))
    np.add.at(out, projector_map(mesh, 0, 7), F(7, uh))
    return out


# ------------------------------------------------------------------ solver ----------------
@dataclass
class History:
    k: int
    res_l2: float
    res_inf: float
    err_max: float
    err_l2: float
    s_hat: float


class SolverContext:
    """SolverContext (solver.hpp:114-155, solver.cpp:486-558)."""

    def __init__(self, mesh: Mesh, prob: Problem, bundle=None):
        self.mesh, self.prob = mesh, prob
        d = mesh.dim
        self.A = assemble_operator(mesh, prob, 0)
        self._bundle = bundle
        self.b = assemble_rhs(mesh, prob, 0) if bundle is None else np.asarray(bundle["fine"], dtype=np.float64)
        self.slab_A = [assemble_operator(mesh, prob, 1 << a) for a in range(d)]
        self.slab_lu = [spla.splu(A.tocsc()) for A in self.slab_A]
        self.coarse_lu = spla.splu(assemble_operator(mesh, prob, (1 << d) - 1).tocsc())
        self.fine_to_slab = [projector_map(mesh, 0, 1 << a) for a in range(d)]
        self.blocks = hole_blocks(mesh)
        blk = self.A[self.blocks[0]][:, self.blocks[0]]
        self.shared = all((self.A[p][:, p] != blk).nnz == 0 for p in self.blocks[1:])  # linsolve.cpp:134-139
        self.hole_lu = [spla.splu(blk.tocsc())] if self.shared else [spla.splu(self.A[p][:, p].tocsc()) for p in self.blocks]

    def assembled_bundle(self):
        if self._bundle is not None:
            return self._bundle
        d = self.mesh.dim
        return {"fine": self.b, "aniso": [assemble_rhs(self.mesh, self.prob, 1 << a) for a in range(d)],
                "coarse": assemble_rhs(self.mesh, self.prob, (1 << d) - 1)}

    def fill(self, skeleton, b):
        """fill_core (solver.cpp:414-432); shared hole factorization solved for all holes at once."""
        out = skeleton.copy()
        Ask = csr_matvec_ordered(self.A, skeleton)
        P = np.stack(self.blocks, axis=1)  # [points-in-hole, hole]
        rhs = (0.0 if b is None else b[P]) - Ask[P]
        if self.shared:
            out[P] = self.hole_lu[0].solve(rhs)
        else:
            for i in range(P.shape[1]):
                out[P[:, i]] = self.hole_lu[i].solve(rhs[:, i])
        return out

    def initial_guess(self, bundle, seed, normalize):
        """SolverContext::initial_guess (solver.cpp:518-548)."""
        d = self.mesh.dim
        sol = [self.slab_lu[a].solve(bundle["aniso"][a]) for a in range(d)]
        coarse = None
        if not normalize:
            coarse = self.coarse_lu.solve(bundle["coarse"])
        else:
            for a in range(d):
                nrm = math.sqrt(float(np.sum(sol[a] * sol[a])))
                if not nrm > 0.0:
                    raise ZeroNormSolution("zero-norm solution cannot be normalized")
                sol[a] = sol[a] / nrm
        if d == 2:
            skel = build_skeleton_2d(self.mesh, sol[1], sol[0], coarse, seed)
        else:
            skel = merge_3d(self.mesh, sol, coarse, seed)
        return self.fill(skel, bundle["fine"])

    def error_guess(self, r, seed):
        """SolverContext::error_guess (solver.cpp:550-558)."""
        bundle = {"fine": None, "aniso": [r[m] for m in self.fine_to_slab]}
        return self.initial_guess(bundle, seed, normalize=True)


def optimal_scaling(A, r, e):
    """optimal_scaling with subsample = 0 (solver.cpp:447-484)."""
    w = csr_matvec_ordered(A, e)
    num, den = float(np.dot(r, w)), float(np.dot(w, w))
    if not den > 0.0:
        return 0.0
    q = num / den
    return q if 0.0 < q else 0.0


def asdsm_iterate(mesh: Mesh, prob: Problem, max_iter=20, seed=0, tol=0.0, stagnation_window=0,
                  stagnation_ratio=0.99, exact=None, bundle=None):
    """asdsm_iterate (solver.cpp:565-680).  `bundle` overrides the assembled right-hand sides."""
    ctx = SolverContext(mesh, prob, bundle)
    A, b = ctx.A, ctx.b
    b_l2 = float(np.linalg.norm(b))
    stop_at = tol * (b_l2 if b_l2 > 0 else 1.0)
    cell = float(np.prod(mesh.h))
    hist: List[History] = []

    def record(k, u, r, s):
        em = el = float("nan")
        if exact is not None:
            dlt = u - exact
            em, el = float(np.max(np.abs(dlt))), math.sqrt(float(np.sum(dlt * dlt)) * cell)
        hist.append(History(k, float(np.linalg.norm(r)), float(np.max(np.abs(r))), em, el, s))

    u = ctx.initial_guess(ctx.assembled_bundle(), mix_seed(seed, 0), normalize=False)
    r = residual(A, b, u)
    record(0, u, r, float("nan"))
    stop = "tol" if hist[-1].res_l2 <= stop_at else ""
    k = 1
    while k <= max_iter and not stop:
        sk = mix_seed(seed, k)
        rn = hist[-1].res_l2
        s = 0.0
        try:
            e = ctx.error_guess(r, sk)
            s = optimal_scaling(A, r, e)
            if s != 0.0:
                un = u + s * e
                rn_vec = residual(A, b, un)
                if float(np.linalg.norm(rn_vec)) > rn * (1.0 + 1e-12):
                    s = 0.0
                else:
                    u, r = un, rn_vec
        except ZeroNormSolution:
            s = 0.0
        record(k, u, r, s)
        if hist[-1].res_l2 <= stop_at:
            stop = "tol"
        elif stagnation_window > 0 and k >= stagnation_window:
            if hist[-1].res_l2 > hist[k - stagnation_window].res_l2 * stagnation_ratio ** stagnation_window:
                stop = "stagnation"
        k += 1
    return u, r, hist, stop or "max_iter"


# ------------------------------------------------------------------ problem catalogue ------
def constant_problem(dim, alpha, beta, time_dependent=False):
    """A constant-coefficient ProblemSpec whose rhs comes from a bundle (source/boundary unused)."""
    al = [(lambda v: (lambda x: np.full(x.shape[1], v)))(float(a)) for a in alpha]
    be = [(lambda v: (lambda x: np.full(x.shape[1], v)))(float(b)) for b in beta]
    zero = lambda x: np.zeros(x.shape[1])  # noqa: E731
    return Problem(dim, al, be, zero, zero, None, time_dependent)


def reference_example(example: int, setting: int) -> Problem:
    """make_problem (problems.cpp:13-141)."""
    pi = math.pi
    one = lambda x: np.ones(x.shape[1])  # noqa: E731
    if example == 1 and setting == 2:  # problems.cpp:27-43
        th = lambda x: 4.0 * pi * (x[0] + x[1])  # noqa: E731
        ex = lambda x: np.sin(4.0 * pi * x[0] + 4.0 * pi * x[1])  # noqa: E731
        return Problem(2, [lambda x: 1.0 + x[0] * x[0], lambda x: 2.0 + x[0] * x[1]],
                       [lambda x: 2.0 - x[0], lambda x: 1.0 + x[1]],
                       lambda x: 16.0 * pi * pi * (3.0 + x[0] * x[0] + x[0] * x[1]) * np.sin(th(x))
                       + 4.0 * pi * (3.0 - x[0] + x[1]) * np.cos(th(x)), ex, ex)
    if example in (1, 2) and setting == 1:
        return Problem(2, [one, one], [one, one],
                       lambda x: 2.0 * pi * pi * np.sin(pi * x[0] + pi * x[1]) + 2.0 * pi * np.cos(pi * x[0] + pi * x[1]),
                       lambda x: np.sin(pi * x[0] + pi * x[1]), lambda x: np.sin(pi * x[0] + pi * x[1]))
    if (example == 3 and setting == 1) or (example == 2 and setting == 2):
        th = lambda x: pi * (x[0] + x[1])  # noqa: E731
        return Problem(2, [one], [one], lambda x: pi * pi * np.sin(th(x)) + 2.0 * pi * np.cos(th(x)),
                       lambda x: np.sin(pi * x[0] + pi * x[1]), lambda x: np.sin(pi * x[0] + pi * x[1]), True)
    if example == 4 and setting == 1:
        th = lambda x: pi * (x[0] + x[1] + x[2])  # noqa: E731
        return Problem(3, [one] * 3, [one] * 3, lambda x: 3.0 * pi * pi * np.sin(th(x)) + 3.0 * pi * np.cos(th(x)),
                       lambda x: np.sin(th(x)), lambda x: np.sin(th(x)))
    raise NotImplementedError("variable-coefficient examples are not restated here")
