"""Helpers to run the compiled reference oracle (oracle/_ref/ref_dump) and load its dumps.

Test infrastructure only: the checker, never the thing measured or shipped.
"""
import os
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DUMP = os.path.join(ROOT, "oracle", "_ref", "ref_dump")


def have_ref():
    return os.path.exists(REF_DUMP)


def _meta(prefix):
    with open(prefix + ".meta.txt") as f:
        lines = f.read().split("\n")
    dim, ta = map(int, lines[0].split())
    nf = list(map(int, lines[1].split()))
    nc = list(map(int, lines[2].split()))
    return dim, ta, nf, nc


def ref_iterate(spec, nf, nc, iters, seed, env=None, extra=None):
    return _ref_iterate_wait(_ref_iterate_start(spec, nf, nc, iters, seed, env, extra))


ORDER_ENV = {"cm": {"ASDSM_STUB_ORDER": "cm"}, "natural": {"ASDSM_STUB_NATURAL_ORDER": "1"}}


def ref_iterate_pair(spec, nf, nc, iters, seed, extra=None, orders=("cm", "natural")):
    """The reference run (reverse Cuthill-McKee fill ordering, as shipped in the Eigen stand-in)
    and the same run under other equally valid fill orderings of its sparse LU (Cuthill-McKee,
    natural), all concurrently: (ref, [alt, ...]).  Eigen's own SparseLU uses yet another one
    (COLAMD); the reference fixes none of them."""
    jobs = [_ref_iterate_start(spec, nf, nc, iters, seed, None, extra)]
    jobs += [_ref_iterate_start(spec, nf, nc, iters, seed, ORDER_ENV[o], extra) for o in orders]
    out = [_ref_iterate_wait(j) for j in jobs]
    return out[0], out[1:]


def reproducibility_floor(ref, alts):
    """Relative spread of the reference's residual history against itself under the other valid
    fill orderings (max over them), made non-decreasing in k (rounding differences propagate)."""
    want = ref["hist"][:, 1]
    spread = np.max([np.abs(a["hist"][:, 1] - want) / want for a in alts], axis=0)
    return np.maximum.accumulate(spread)


def history_tolerance(ref, alts):
    """Per-iteration absolute bound on |res_l2(gpu) - res_l2(ref)|: relative 1e-10 where the
    reference reproduces itself to 1e-10, else 10x its own ordering spread (DESIGN.md Parity)."""
    want = ref["hist"][:, 1]
    return want * np.maximum(1e-10, 10.0 * reproducibility_floor(ref, alts))


def _ref_iterate_start(spec, nf, nc, iters, seed, env=None, extra=None):
    d = tempfile.TemporaryDirectory()
    prefix = os.path.join(d.name, "run")
    e = dict(os.environ)
    if env:
        e.update(env)
    p = subprocess.Popen([REF_DUMP, "iterate", spec, str(nf), str(nc), str(iters), str(seed), prefix]
                         + list(extra or []), env=e, stdout=subprocess.DEVNULL)
    return p, d, prefix


def _ref_iterate_wait(job):
    p, d, prefix = job
    with d:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, p.args)
        rows = []
        stop = None
        with open(prefix + ".hist.txt") as f:
            for line in f:
                if line.startswith("# stop:"):
                    stop = line.split(":")[1].strip()
                    continue
                rows.append([float(x) for x in line.split()])
        out = {
            "hist": np.array(rows),
            "stop": stop,
            "u": np.fromfile(prefix + ".u.f64"),
            "r": np.fromfile(prefix + ".r.f64"),
            "u0": np.fromfile(prefix + ".u0.f64"),
            "r0": np.fromfile(prefix + ".r0.f64"),
            "meta": _meta(prefix),
        }
    return out


def ref_bundle(spec, nf, nc):
    with tempfile.TemporaryDirectory() as d:
        prefix = os.path.join(d, "b")
        subprocess.check_call([REF_DUMP, "bundle", spec, str(nf), str(nc), prefix])
        dim, ta, fnf, fnc = _meta(prefix)
        out = {"meta": (dim, ta, fnf, fnc), "fine": np.fromfile(prefix + ".b_fine.f64"),
               "aniso": [np.fromfile(prefix + f".b_slab{a}.f64") for a in range(dim)],
               "coarse": np.fromfile(prefix + ".b_coarse.f64"),
               "A_rowptr": np.fromfile(prefix + ".A_rowptr.i64", dtype=np.int64),
               "A_col": np.fromfile(prefix + ".A_col.i64", dtype=np.int64),
               "A_val": np.fromfile(prefix + ".A_val.f64")}
        if os.path.exists(prefix + ".exact.f64"):
            out["exact"] = np.fromfile(prefix + ".exact.f64")
    return out


def ref_error_guess(spec, nf, nc, seed, r):
    with tempfile.TemporaryDirectory() as d:
        rfile = os.path.join(d, "r.f64")
        np.asarray(r, dtype=np.float64).tofile(rfile)
        prefix = os.path.join(d, "eg")
        subprocess.check_call([REF_DUMP, "errguess", spec, str(nf), str(nc), str(seed), rfile, prefix])
        e = np.fromfile(prefix + ".e.f64")
        with open(prefix + ".s.txt") as f:
            s = float(f.read())
    return e, s


def ref_maps(spec, nf, nc):
    with tempfile.TemporaryDirectory() as d:
        prefix = os.path.join(d, "m")
        subprocess.check_call([REF_DUMP, "maps", spec, str(nf), str(nc), prefix])
        dim = _meta(prefix)[0]
        maps = {}
        full = (1 << dim) - 1
        for fr in range(full + 1):
            for to in range(full + 1):
                if fr == to or (fr & to) != fr:
                    continue
                maps[(fr, to)] = np.fromfile(prefix + f".map_{fr}_{to}.i64", dtype=np.int64)
        maps["holes"] = np.fromfile(prefix + ".map_holes.i64", dtype=np.int64)
    return maps


def csr_residual_exact(bundle, u, b=None):
    """b - A u with the reference's CSR row order (sparse.cpp:49-58), vectorized per column slot.

    Each row's entries are summed left to right starting from 0.0 exactly as the reference does,
    so the result is bitwise the reference's residual.
    """
    rp, col, val = bundle["A_rowptr"], bundle["A_col"], bundle["A_val"]
    n = len(rp) - 1
    b = bundle["fine"] if b is None else b
    counts = np.diff(rp)
    acc = np.zeros(n)
    for slot in range(int(counts.max())):
        rows = np.nonzero(counts > slot)[0]
        idx = rp[rows] + slot
        acc[rows] = acc[rows] + val[idx] * u[col[idx]]
    return b - acc


def eval_floor(bundle, u):
    """fp64 evaluation floor of the residual: eps * || |A| |u| ||_2 (A from the reference CSR)."""
    rp, col, val = bundle["A_rowptr"], bundle["A_col"], bundle["A_val"]
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    absau = np.zeros(n)
    np.add.at(absau, rows, np.abs(val) * np.abs(u[col]))
    return np.finfo(np.float64).eps * float(np.linalg.norm(absau))
