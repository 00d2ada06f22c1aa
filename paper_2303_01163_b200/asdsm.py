"""ctypes mirror of the reference's solver interface over libasdsm_b200.so.

Reference interfaces mirrored (names, argument meaning, error classes):
  MeshKind / MeshConfig        proj/include/asdsm/mesh.hpp:22-83
  build_projector / hole_blocks proj/include/asdsm/mesh.hpp:148-154
  make_problem                  proj/include/asdsm/problems.hpp:20
  SolverContext                 proj/include/asdsm/solver.hpp:114-155
  IterateOptions, IterationState, asdsm_iterate  proj/include/asdsm/solver.hpp:44-163
  error classes                 proj/include/asdsm/errors.hpp:8-66
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))


class Error(RuntimeError):
    """asdsm::Error (errors.hpp:9)."""


class DivisibilityError(Error):
    pass


class DegenerateError(Error):
    pass


class IndexOutOfRange(Error):
    pass


class NotASubmesh(Error):
    pass


class InvalidKind(Error):
    pass


class DimensionMismatch(Error):
    pass


class SingularMatrix(Error):
    pass


class SkeletonNotHollow(Error):
    pass


class ZeroNormSolution(Error):
    pass


class UnknownExample(Error):
    pass


class NoExactSolution(Error):
    pass


class Unsupported(Error):
    """A configuration outside the B200 path's scope (e.g. variable coefficients)."""


class CudaFailure(Error):
    pass


_CODES = {
    1: Error, 2: DivisibilityError, 3: DegenerateError, 4: IndexOutOfRange, 5: NotASubmesh,
    6: InvalidKind, 7: DimensionMismatch, 8: SingularMatrix, 9: SkeletonNotHollow,
    10: ZeroNormSolution, 11: UnknownExample, 12: NoExactSolution, 13: Unsupported, 14: CudaFailure,
}
_STOP = {1: "tol", 2: "stagnation", 3: "max_iter"}

_lib = None


def library_path() -> str:
    # ASDSM_LIB: an instrumented build of the same library (profiling only)
    return os.environ.get("ASDSM_LIB") or os.path.join(_HERE, "libasdsm_b200.so")


_FIELD_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p)


class _Field(ctypes.Structure):
    _fields_ = [("fn", _FIELD_FN), ("ctx", ctypes.c_void_p)]


class _ProblemSpec(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("time_dependent", ctypes.c_int32), ("alpha", _Field * 3),
                ("beta", _Field * 3), ("source", _Field), ("boundary", _Field), ("exact", _Field)]


_OBSERVER_FN = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_void_p)


class _Options(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iter", ctypes.c_int32),
                ("stagnation_window", ctypes.c_int32), ("stagnation_ratio", ctypes.c_double),
                ("subsample", ctypes.c_double), ("rng_seed", ctypes.c_uint64), ("sparse_residual", ctypes.c_int32)]


def load_library():
    """Load the in-tree libasdsm_b200.so; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    I = ctypes.c_int
    D = ctypes.POINTER(ctypes.c_double)
    IP = ctypes.POINTER(ctypes.c_int)
    I64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "asdsm_last_error": (ctypes.c_char_p, []),
        "asdsm_abi_version": (I, []),
        "asdsm_problem_example": (I, [I, I, ctypes.POINTER(P)]),
        "asdsm_problem_config": (I, [I, ctypes.c_uint64, ctypes.POINTER(P)]),
        "asdsm_problem_create": (I, [ctypes.POINTER(_ProblemSpec), ctypes.POINTER(P)]),
        "asdsm_problem_destroy": (None, [P]),
        "asdsm_problem_info": (I, [P, IP, IP, IP, D, D, IP]),
        "asdsm_config_mesh": (I, [I, IP, IP, IP, IP, IP]),
        "asdsm_assemble_rhs": (I, [P, I, IP, IP, I, ctypes.c_uint, D]),
        "asdsm_sample_exact": (I, [P, I, IP, IP, I, D]),
        "asdsm_plan_create": (I, [I, IP, IP, I, D, D, ctypes.POINTER(P)]),
        "asdsm_plan_destroy": (None, [P]),
        "asdsm_plan_create_problem": (I, [P, I, IP, IP, I, ctypes.POINTER(P)]),
        "asdsm_plan_is_variable": (I, [P]),
        "asdsm_point_count": (I, [P, ctypes.c_uint, I, I64]),
        "asdsm_projector_map": (I, [P, ctypes.c_uint, ctypes.c_uint, I, I64]),
        "asdsm_set_bundle": (I, [P, D, ctypes.POINTER(D), D, D, I]),
        "asdsm_set_bundle_async": (I, [P, D, ctypes.POINTER(D), D, D, I, P]),
        "asdsm_iterate": (I, [P, ctypes.POINTER(_Options), D, IP, IP, D, D]),
        "asdsm_iterate_async": (I, [P, ctypes.POINTER(_Options), P]),
        "asdsm_iterate_observed": (I, [P, ctypes.POINTER(_Options), _OBSERVER_FN, P, D, IP, IP, D, D]),
        "asdsm_fetch": (I, [P, P, D, IP, IP, D, D]),
        "asdsm_solve": (I, [P, D, ctypes.POINTER(D), D, D, ctypes.POINTER(_Options), D, IP, IP, D, D]),
        "asdsm_device_solution": (I, [P, P, ctypes.POINTER(ctypes.c_void_p)]),
        "asdsm_last_launch_count": (ctypes.c_int64, [P]),
        "asdsm_plan_kernels": (I, [P, ctypes.c_char_p, ctypes.c_int64]),
        "asdsm_residual": (I, [P, D, D, D]),
        "asdsm_initial_guess": (I, [P, D]),
        "asdsm_error_guess": (I, [P, D, ctypes.c_uint64, D]),
        "asdsm_optimal_scaling": (I, [P, D, D, D]),
        "asdsm_richardson_extrapolate": (I, [P, D, D, D, D]),
        "asdsm_choose_cross_points": (I, [P, D, D, ctypes.c_uint64, D]),
        "asdsm_spline_correct": (I, [P, D, D, I, D]),
        "asdsm_build_skeleton": (I, [P, D, D, D, I, ctypes.c_uint64, D]),
        "asdsm_merge_3d": (I, [P, D, D, D, D, ctypes.c_uint64, D]),
        "asdsm_fill_holes": (I, [P, D, D, D]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int):
    if rc != 0:
        msg = load_library().asdsm_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i32(seq: Sequence[int], n: int = 3):
    arr = (ctypes.c_int * n)()
    for i, v in enumerate(seq):
        arr[i] = int(v)
    return arr


def _d3(seq: Sequence[float]):
    arr = (ctypes.c_double * 3)()
    for i, v in enumerate(seq):
        arr[i] = float(v)
    return arr


# ---------------------------------------------------------------- mesh (mesh.hpp) -----------
@dataclass(frozen=True)
class MeshKind:
    """A tensor mesh kind (coarse mask) or the holes set (mesh.hpp:22-54)."""
    dim: int
    mask: int = 0
    holes: bool = False

    @staticmethod
    def fine(dim):
        return MeshKind(dim, 0, False)

    @staticmethod
    def coarse(dim):
        return MeshKind(dim, (1 << dim) - 1, False)

    @staticmethod
    def holes_of(dim):
        return MeshKind(dim, 0, True)

    @staticmethod
    def coarse_along(dim, axis):
        if dim < 2 or dim > 3:
            raise DimensionMismatch(f"mesh dimension must be 2 or 3, got {dim}")
        if axis < 0 or axis >= dim:
            raise IndexOutOfRange(f"coarse_along: axis {axis}")
        return MeshKind(dim, 1 << axis, False)

    @staticmethod
    def from_mask(dim, mask):
        if mask >= (1 << dim):
            raise IndexOutOfRange("from_mask: mask out of range")
        return MeshKind(dim, mask, False)

    def coarse_on(self, axis):
        return (not self.holes) and bool((self.mask >> axis) & 1)

    def name(self):
        if self.holes:
            return "[holes]"
        return "[" + ",".join("H" if self.coarse_on(a) else "h" for a in range(self.dim)) + "]"


@dataclass
class MeshConfig:
    """MeshConfig (mesh.hpp:56-83); validation mirrors MeshConfig::create (mesh.cpp:47-76)."""
    dim: int
    fine_counts: List[int]
    coarse_counts: List[int]
    factors: List[int]
    fine_steps: List[float]
    coarse_steps: List[float]
    time_axis: int = -1

    @staticmethod
    def create(dim, fine_counts, coarse_counts, time_axis=-1):
        if dim < 2 or dim > 3:
            raise DimensionMismatch(f"mesh dimension must be 2 or 3, got {dim}")
        if len(fine_counts) != dim or len(coarse_counts) != dim:
            raise DimensionMismatch("mesh counts must have one entry per axis")
        if time_axis not in (-1, dim - 1):
            raise DimensionMismatch("time axis must be the last axis")
        factors, fs, cs = [], [], []
        for a in range(dim):
            nf, nc = int(fine_counts[a]), int(coarse_counts[a])
            if nf < 1 or nc < 1:
                raise DegenerateError(f"axis {a}: interior point counts must be >= 1")
            if (nf + 1) % (nc + 1) != 0:
                raise DivisibilityError(f"axis {a}: fine intervals {nf + 1} not divisible by coarse intervals {nc + 1}")
            n = (nf + 1) // (nc + 1)
            if n < 2:
                raise DegenerateError(f"axis {a}: refinement factor 1 leaves no holes")
            factors.append(n)
            fs.append(1.0 / float(nf + 1))
            cs.append(float(n) * (1.0 / float(nf + 1)))
        return MeshConfig(dim, [int(x) for x in fine_counts], [int(x) for x in coarse_counts], factors, fs, cs,
                          time_axis)

    def axis_points(self, kind: MeshKind, axis: int) -> int:
        if kind.holes:
            raise InvalidKind("holes mesh has no per-axis point count")
        return self.coarse_counts[axis] if kind.coarse_on(axis) else self.fine_counts[axis]

    def point_count(self, kind: MeshKind) -> int:
        if kind.holes:
            n = 1
            for a in range(self.dim):
                n *= (self.coarse_counts[a] + 1) * (self.factors[a] - 1)
            return n
        n = 1
        for a in range(self.dim):
            n *= self.axis_points(kind, a)
        return n

    def shape(self, kind: MeshKind):
        """numpy shape (slowest axis first) of a kind's x-fastest layout."""
        return tuple(self.axis_points(kind, a) for a in reversed(range(self.dim)))


# ---------------------------------------------------------------- problems ------------------
class Problem:
    """Handle on a ProblemSpec of the library's catalogue (problems.hpp:20 + BASELINE configs)."""

    def __init__(self, handle, label):
        self._h = handle
        self.label = label
        lib = load_library()
        dim, td, cc, he = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        al, be = (ctypes.c_double * 3)(), (ctypes.c_double * 3)()
        _check(lib.asdsm_problem_info(self._h, ctypes.byref(dim), ctypes.byref(td), ctypes.byref(cc), al, be,
                                      ctypes.byref(he)))
        self.dim = dim.value
        self.time_dependent = bool(td.value)
        self.constant_coeffs = bool(cc.value)
        self.alpha = list(al)
        self.beta = list(be)
        self.has_exact = bool(he.value)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.asdsm_problem_destroy(self._h)
            self._h = None

    def assemble_rhs(self, config: MeshConfig, kind: MeshKind) -> np.ndarray:
        """assemble_rhs (fdm.hpp:44-46), host-side sampling."""
        if kind.holes:
            raise InvalidKind("holes have no standalone right-hand side")
        out = np.empty(config.point_count(kind), dtype=np.float64)
        _check(load_library().asdsm_assemble_rhs(self._h, config.dim, _i32(config.fine_counts),
                                                 _i32(config.coarse_counts), config.time_axis, kind.mask, _dptr(out)))
        return out

    def sample_exact(self, config: MeshConfig) -> np.ndarray:
        out = np.empty(config.point_count(MeshKind.fine(config.dim)), dtype=np.float64)
        _check(load_library().asdsm_sample_exact(self._h, config.dim, _i32(config.fine_counts),
                                                 _i32(config.coarse_counts), config.time_axis, _dptr(out)))
        return out


class ProblemSpec:
    """The reference's ProblemSpec (fdm.hpp:17-30) with caller-defined fields: Python callables
    f(x) of a point x (a sequence of `dim` floats; the last one is t when time_dependent).
    alpha / beta hold one callable per spatial axis.  The fields are evaluated on the host while
    a plan is built and its right-hand sides assembled (asdsm_problem_create), never during a
    solve; `problem()` returns the library handle (a Problem) usable wherever a catalogue
    problem is."""

    def __init__(self, dim: int, alpha, beta, source, boundary, exact=None, time_dependent: bool = False):
        self.dim = int(dim)
        self.time_dependent = bool(time_dependent)
        self.alpha = list(alpha)
        self.beta = list(beta)
        self.source = source
        self.boundary = boundary
        self.exact = exact

    def spatial_axes(self) -> int:
        return self.dim - 1 if self.time_dependent else self.dim

    def problem(self) -> "Problem":
        lib = load_library()
        dim = self.dim
        keep = []

        def field(f):
            if f is None:
                return _Field(_FIELD_FN(), None)

            def tramp(x, _ctx, f=f):
                return float(f(tuple(x[a] for a in range(dim))))
            cb = _FIELD_FN(tramp)
            keep.append(cb)
            return _Field(cb, None)

        spec = _ProblemSpec()
        spec.dim = dim
        spec.time_dependent = int(self.time_dependent)
        for a in range(self.spatial_axes()):
            spec.alpha[a] = field(self.alpha[a])
            spec.beta[a] = field(self.beta[a])
        spec.source = field(self.source)
        spec.boundary = field(self.boundary)
        spec.exact = field(self.exact)
        h = ctypes.c_void_p()
        _check(lib.asdsm_problem_create(ctypes.byref(spec), ctypes.byref(h)))
        prob = Problem(h, "caller-defined ProblemSpec")
        prob._keep = keep  # the callbacks live as long as the handle
        return prob


def make_problem(example: int, setting: int) -> Problem:
    """make_problem (problems.hpp:20, problems.cpp:114-141)."""
    lib = load_library()
    h = ctypes.c_void_p()
    _check(lib.asdsm_problem_example(int(example), int(setting), ctypes.byref(h)))
    return Problem(h, f"example {example} setting {setting}")


def baseline_problem(config_id: int, seed: int = 0) -> Problem:
    lib = load_library()
    h = ctypes.c_void_p()
    _check(lib.asdsm_problem_config(int(config_id), ctypes.c_uint64(seed), ctypes.byref(h)))
    return Problem(h, f"config {config_id} seed {seed}")


def baseline_mesh(config_id: int):
    """(MeshConfig, iterations) of a BASELINE.json config (see DESIGN.md for the mesh rule)."""
    lib = load_library()
    dim, ta, it = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    nf, nc = (ctypes.c_int * 3)(), (ctypes.c_int * 3)()
    _check(lib.asdsm_config_mesh(int(config_id), ctypes.byref(dim), nf, nc, ctypes.byref(ta), ctypes.byref(it)))
    d = dim.value
    return MeshConfig.create(d, list(nf)[:d], list(nc)[:d], ta.value), it.value


def example_mesh(example: int, setting: int, nf: int, nc: int) -> MeshConfig:
    """example_mesh (problems.hpp:23)."""
    p = make_problem(example, setting)
    return MeshConfig.create(p.dim, [nf] * p.dim, [nc] * p.dim, p.dim - 1 if p.time_dependent else -1)


# ---------------------------------------------------------------- solver --------------------
@dataclass
class IterateOptions:
    """IterateOptions (solver.hpp:56-68)."""
    tol: float = 1e-12
    max_iter: int = 20
    stagnation_window: int = 3
    stagnation_ratio: float = 0.99
    subsample: float = 0.0
    rng_seed: int = 0
    sparse_residual: bool = False
    # called with the IterationState after each recorded iteration (k = 0 first), as
    # solver.hpp:65-66 (C-ABI asdsm_iterate_observed: launch by launch, one sync per iteration)
    observer: Optional[Callable[["IterationState"], None]] = None

    def _c(self):
        return _Options(self.tol, self.max_iter, self.stagnation_window, self.stagnation_ratio, self.subsample,
                        self.rng_seed, int(self.sparse_residual))


@dataclass
class IterationRecord:
    k: int
    res_l2: float
    res_inf: float
    err_max: float
    err_l2: float
    s_hat: float
    wall_ms: float


@dataclass
class IterationState:
    u: np.ndarray
    r: np.ndarray
    history: List[IterationRecord] = field(default_factory=list)
    stop_reason: str = ""


class SolverContext:
    """SolverContext (solver.hpp:114-155): device-resident operators, rhs bundle, tables."""

    def __init__(self, config: MeshConfig, problem: Problem, bundle=None):
        if problem.dim != config.dim:
            raise DimensionMismatch("problem/mesh dimension mismatch")
        if problem.time_dependent != (config.time_axis >= 0):
            raise DimensionMismatch("problem and mesh disagree about a time axis")
        self.config = config
        self.problem = problem
        lib = load_library()
        self._lib = lib
        h = ctypes.c_void_p()
        _check(lib.asdsm_plan_create_problem(problem._h, config.dim, _i32(config.fine_counts),
                                             _i32(config.coarse_counts), config.time_axis, ctypes.byref(h)))
        self._h = h
        self.bundle = bundle if bundle is not None else self.assembled_bundle()
        self.exact = problem.sample_exact(config) if problem.has_exact else None
        self.set_bundle(self.bundle, self.exact)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.asdsm_plan_destroy(self._h)
            self._h = None

    def assembled_bundle(self):
        """assembled_bundle (solver.hpp:125): fine, per-axis anisotropic, coarse rhs."""
        c, p = self.config, self.problem
        fine = p.assemble_rhs(c, MeshKind.fine(c.dim))
        aniso = [p.assemble_rhs(c, MeshKind.coarse_along(c.dim, a)) for a in range(c.dim)]
        coarse = p.assemble_rhs(c, MeshKind.coarse(c.dim))
        return {"fine": fine, "aniso": aniso, "coarse": coarse}

    def set_bundle(self, bundle, exact=None):
        slabs = (ctypes.POINTER(ctypes.c_double) * 3)()
        keep = [np.ascontiguousarray(x, dtype=np.float64) for x in bundle["aniso"]]
        for a, x in enumerate(keep):
            slabs[a] = _dptr(x)
        fine = np.ascontiguousarray(bundle["fine"], dtype=np.float64)
        coarse = np.ascontiguousarray(bundle["coarse"], dtype=np.float64)
        ex = None if exact is None else np.ascontiguousarray(exact, dtype=np.float64)
        _check(self._lib.asdsm_set_bundle(self._h, _dptr(fine), slabs, _dptr(coarse), _dptr(ex), 0))

    def fine_size(self):
        return self.config.point_count(MeshKind.fine(self.config.dim))

    def residual(self, u: np.ndarray, b: Optional[np.ndarray] = None) -> np.ndarray:
        """residual (fdm.hpp:50): b - A_ff u."""
        b = self.bundle["fine"] if b is None else b
        u = np.ascontiguousarray(u, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        r = np.empty_like(u)
        _check(self._lib.asdsm_residual(self._h, _dptr(u), _dptr(b), _dptr(r)))
        return r

    def initial_guess(self) -> np.ndarray:
        """initial_guess with the assembled bundle (smooth mode, solver.hpp:132)."""
        u = np.empty(self.fine_size(), dtype=np.float64)
        _check(self._lib.asdsm_initial_guess(self._h, _dptr(u)))
        return u

    def error_guess(self, r: np.ndarray, seed: int) -> np.ndarray:
        """error_guess (solver.hpp:135)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        e = np.empty_like(r)
        _check(self._lib.asdsm_error_guess(self._h, _dptr(r), ctypes.c_uint64(seed), _dptr(e)))
        return e

    def optimal_scaling(self, r: np.ndarray, e: np.ndarray) -> float:
        """optimal_scaling with subsample = 0 (solver.hpp:109)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        s = ctypes.c_double()
        _check(self._lib.asdsm_optimal_scaling(self._h, _dptr(r), _dptr(e), ctypes.byref(s)))
        return s.value

    def iterate(self, options: IterateOptions = IterateOptions()) -> IterationState:
        n = self.fine_size()
        u = np.empty(n, dtype=np.float64)
        r = np.empty(n, dtype=np.float64)
        hist = np.empty((max(options.max_iter, 0) + 1) * 7, dtype=np.float64)
        nrec, stop = ctypes.c_int(), ctypes.c_int()
        opts = options._c()
        if options.observer is None:
            _check(self._lib.asdsm_iterate(self._h, ctypes.byref(opts), _dptr(hist), ctypes.byref(nrec),
                                           ctypes.byref(stop), _dptr(u), _dptr(r)))
        else:
            def seen(hp, nr, up, rp, nn, _ctx):
                h = np.ctypeslib.as_array(hp, shape=(max(nr, 1) * 7,))[: nr * 7].reshape(-1, 7)
                options.observer(IterationState(
                    np.ctypeslib.as_array(up, shape=(nn,)).copy(), np.ctypeslib.as_array(rp, shape=(nn,)).copy(),
                    [IterationRecord(int(x[0]), x[1], x[2], x[3], x[4], x[5], x[6]) for x in h], ""))
            cb = _OBSERVER_FN(seen)
            _check(self._lib.asdsm_iterate_observed(self._h, ctypes.byref(opts), cb, None, _dptr(hist),
                                                    ctypes.byref(nrec), ctypes.byref(stop), _dptr(u), _dptr(r)))
        rows = hist[: nrec.value * 7].reshape(-1, 7)
        history = [IterationRecord(int(x[0]), x[1], x[2], x[3], x[4], x[5], x[6]) for x in rows]
        return IterationState(u, r, history, _STOP.get(stop.value, "max_iter"))

    def solve(self, bundle, exact=None, options: IterateOptions = IterateOptions(), u_out=None,
              r_out=None) -> IterationState:
        """New right-hand sides + asdsm_iterate in one call (C-ABI asdsm_solve: the uploads, the
        solve and the downloads on the plan's stream, one synchronize).  u_out / r_out: optional
        float64 host arrays (e.g. pinned) the final iterate and residual are written to."""
        n = self.fine_size()
        u = np.empty(n, dtype=np.float64) if u_out is None else u_out
        r = np.empty(n, dtype=np.float64) if r_out is None else r_out
        slabs = (ctypes.POINTER(ctypes.c_double) * 3)()
        keep = [np.ascontiguousarray(x, dtype=np.float64) for x in bundle["aniso"]]
        for a, x in enumerate(keep):
            slabs[a] = _dptr(x)
        fine = np.ascontiguousarray(bundle["fine"], dtype=np.float64)
        coarse = np.ascontiguousarray(bundle["coarse"], dtype=np.float64)
        ex = None if exact is None else np.ascontiguousarray(exact, dtype=np.float64)
        hist = np.empty((max(options.max_iter, 0) + 1) * 7, dtype=np.float64)
        nrec, stop = ctypes.c_int(), ctypes.c_int()
        opts = options._c()
        _check(self._lib.asdsm_solve(self._h, _dptr(fine), slabs, _dptr(coarse), _dptr(ex), ctypes.byref(opts),
                                     _dptr(hist), ctypes.byref(nrec), ctypes.byref(stop), _dptr(u), _dptr(r)))
        self.bundle, self.exact = bundle, exact
        rows = hist[: nrec.value * 7].reshape(-1, 7)
        history = [IterationRecord(int(x[0]), x[1], x[2], x[3], x[4], x[5], x[6]) for x in rows]
        return IterationState(u, r, history, _STOP.get(stop.value, "max_iter"))

    # ---- the reference's public solver stages (solver.hpp:70-105) on this plan's mesh ----------
    def _kind_len(self, mask: int) -> int:
        return self.config.point_count(MeshKind.from_mask(self.config.dim, mask))

    def _in(self, a, mask):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.size != self._kind_len(mask):
            raise DimensionMismatch("stage input has the wrong point count for its mesh kind")
        return a

    def richardson_extrapolate(self, u1_cc, u2_cc, u_cc) -> np.ndarray:
        full = (1 << self.config.dim) - 1
        ins = [self._in(x, full) for x in (u1_cc, u2_cc, u_cc)]
        out = np.empty(self._kind_len(full))
        _check(self._lib.asdsm_richardson_extrapolate(self._h, *[_dptr(x) for x in ins], _dptr(out)))
        return out

    def choose_cross_points(self, u_fc, u_cf, rng_seed: int = 0) -> np.ndarray:
        a, b = self._in(u_fc, 2), self._in(u_cf, 1)
        out = np.empty(self._kind_len(3))
        _check(self._lib.asdsm_choose_cross_points(self._h, _dptr(a), _dptr(b), ctypes.c_uint64(rng_seed), _dptr(out)))
        return out

    def spline_correct(self, u_aniso, e_cc, dense_axis: int) -> np.ndarray:
        if not 0 <= dense_axis <= 1:
            raise IndexOutOfRange("dense_axis must be 0 or 1")
        mask = 1 << (1 - dense_axis)
        a, e = self._in(u_aniso, mask), self._in(e_cc, 3)
        out = np.empty(a.size)
        _check(self._lib.asdsm_spline_correct(self._h, _dptr(a), _dptr(e), int(dense_axis), _dptr(out)))
        return out

    def build_skeleton(self, u_fc, u_cf, u_cc=None, normalized: bool = False, rng_seed: int = 0) -> np.ndarray:
        a, b = self._in(u_fc, 2), self._in(u_cf, 1)
        c = None if u_cc is None else self._in(u_cc, 3)
        out = np.empty(self.fine_size())
        _check(self._lib.asdsm_build_skeleton(self._h, _dptr(a), _dptr(b), _dptr(c), int(bool(normalized)),
                                              ctypes.c_uint64(rng_seed), _dptr(out)))
        return out

    def merge_3d(self, u_x, u_y, u_z, u_ccc=None, rng_seed: int = 0) -> np.ndarray:
        ins = [self._in(x, 1 << a) for a, x in enumerate((u_x, u_y, u_z))]
        c = None if u_ccc is None else self._in(u_ccc, 7)
        out = np.empty(self.fine_size())
        _check(self._lib.asdsm_merge_3d(self._h, *[_dptr(x) for x in ins], _dptr(c), ctypes.c_uint64(rng_seed),
                                        _dptr(out)))
        return out

    def fill_holes(self, skeleton, b_fine=None) -> np.ndarray:
        sk = self._in(skeleton, 0)
        b = None if b_fine is None else self._in(b_fine, 0)
        out = np.empty(sk.size)
        _check(self._lib.asdsm_fill_holes(self._h, _dptr(sk), _dptr(b), _dptr(out)))
        return out

    def variable(self) -> bool:
        """True when the plan runs the variable-coefficient (block-Thomas) path."""
        return bool(self._lib.asdsm_plan_is_variable(self._h))

    def launch_count(self) -> int:
        return int(self._lib.asdsm_last_launch_count(self._h))

    def kernels(self) -> dict:
        """{demangled kernel name: graph nodes} of the last captured solve graph."""
        buf = ctypes.create_string_buffer(1 << 16)
        _check(self._lib.asdsm_plan_kernels(self._h, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, _, n = line.rpartition("\t")
            out[name] = int(n)
        return out

    def projector_map(self, from_kind: MeshKind, to_kind: MeshKind) -> np.ndarray:
        return build_projector(self.config, from_kind, to_kind, plan=self)


def asdsm_iterate(problem: Problem, config: MeshConfig, options: IterateOptions = IterateOptions()) -> IterationState:
    """asdsm_iterate (solver.hpp:161-163)."""
    return SolverContext(config, problem).iterate(options)


def build_projector(config: MeshConfig, from_kind: MeshKind, to_kind: MeshKind, plan: SolverContext = None):
    """build_projector(...).index_map() (mesh.hpp:148), generated by a GPU kernel."""
    if from_kind.holes:
        raise NotASubmesh("cannot project from the holes set")
    if to_kind.holes:
        if from_kind.mask != 0:
            raise NotASubmesh("holes are a subset of the fine mesh only")
    elif (from_kind.mask & to_kind.mask) != from_kind.mask:
        raise NotASubmesh(f"{to_kind.name()} is not a sub-mesh of {from_kind.name()}")
    lib = load_library()
    owned = None
    if plan is None:
        h = ctypes.c_void_p()
        _check(lib.asdsm_plan_create(config.dim, _i32(config.fine_counts), _i32(config.coarse_counts),
                                     config.time_axis, _d3([1, 1, 1]), _d3([0, 0, 0]), ctypes.byref(h)))
        owned = h
        handle = h
    else:
        handle = plan._h
    try:
        out = np.empty(config.point_count(to_kind), dtype=np.int64)
        _check(lib.asdsm_projector_map(handle, from_kind.mask, to_kind.mask, int(to_kind.holes),
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out
    finally:
        if owned is not None:
            lib.asdsm_plan_destroy(owned)


def hole_positions(config: MeshConfig, plan: SolverContext = None) -> np.ndarray:
    """Concatenated hole_blocks positions (mesh.hpp:150-154) = the holes projector map."""
    return build_projector(config, MeshKind.fine(config.dim), MeshKind.holes_of(config.dim), plan)


def nan_to_none(x):
    return None if (x is None or math.isnan(x)) else x


# ---------------------------------------------------------------- runner (runner.hpp) -------
@dataclass
class RunConfig:
    """RunConfig (proj/include/asdsm/runner.hpp:16-27)."""
    example: int = 1
    setting: int = 1
    nf: int = 99
    nc: int = 9
    tol: float = 1e-12
    max_iter: int = 20
    subsample: float = 0.0
    seed: int = 0
    out: str = ""


@dataclass
class RunResult:
    state: IterationState
    csv: str


def _g17(v: float) -> str:
    return "%.17g" % v


def format_history_csv(history: Sequence[IterationRecord]) -> str:
    """format_history_csv (runner.hpp:37, runner.cpp:34-46): fixed header, %.17g floats."""
    lines = ["k,res_l2,res_inf,err_max,err_l2,s_hat,wall_ms"]
    for h in history:
        lines.append(",".join([str(int(h.k))] + [_g17(v) for v in (h.res_l2, h.res_inf, h.err_max, h.err_l2,
                                                                     h.s_hat, h.wall_ms)]))
    return "\n".join(lines) + "\n"


def write_text_file(path: str, content: str):
    """write_text_file (runner.hpp:50)."""
    try:
        with open(path, "w", newline="") as f:
            f.write(content)
    except OSError as e:
        raise Error(f"cannot write {path}") from e


def run_experiment(config: RunConfig) -> RunResult:
    """run_experiment (runner.hpp:41, runner.cpp:48-56)."""
    mesh = example_mesh(config.example, config.setting, config.nf, config.nc)
    prob = make_problem(config.example, config.setting)
    opts = IterateOptions(tol=config.tol, max_iter=config.max_iter, subsample=config.subsample,
                          rng_seed=config.seed)
    st = asdsm_iterate(prob, mesh, opts)
    csv = format_history_csv(st.history)
    if config.out:
        write_text_file(config.out, csv)
    return RunResult(st, csv)


def residual_snapshot(config: RunConfig, at_iter: int) -> str:
    """residual_snapshot (runner.hpp:46, runner.cpp:58-83): |r| after exactly at_iter
    iterations, one CSV row per axis-1 line.  2D meshes only."""
    if at_iter < 0 or at_iter > config.max_iter:
        raise Error(f"snapshot iteration {at_iter} outside [0, max_iter]")
    mesh = example_mesh(config.example, config.setting, config.nf, config.nc)
    if mesh.dim != 2:
        raise DimensionMismatch("residual snapshots need a 2D mesh")
    prob = make_problem(config.example, config.setting)
    opts = IterateOptions(tol=0.0, max_iter=at_iter, stagnation_window=0, subsample=config.subsample,
                          rng_seed=config.seed)
    st = asdsm_iterate(prob, mesh, opts)
    n0, n1 = mesh.fine_counts
    r = np.abs(st.r).reshape(n1, n0)
    return "".join(",".join(_g17(v) for v in row) + "\n" for row in r)
