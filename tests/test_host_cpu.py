"""CPU suite: the C-ABI library and the host side (no GPU compute).

- libasdsm_b200.so loads and exports every entry point include/asdsm_b200.h declares;
- host-side right-hand-side assembly is bitwise the reference's (fdm.cpp:128-171);
- mesh validation / error classes mirror the reference (mesh.cpp:47-76, errors.hpp);
- without a GPU every solve fails loudly (no CPU fallback);
- the multi-rank timing reduction of bench.py (gloo, world_size 2).
"""
import ctypes
import os
import re
import socket
import sys

import numpy as np
import pytest

import paper_2303_01163_b200 as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "asdsm_b200.h")).read()
    names = set(re.findall(r"\b(asdsm_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 20
    lib = ctypes.CDLL(pb.library_path())
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert pb.load_library().asdsm_abi_version() == 4


@pytest.mark.parametrize("name", ["ex1s1_24_4", "ex3s1_24_4", "ex4s1_14_4", "cfg1_49_4", "cfg2_49_4", "cfg3_14_4",
                                  "cfg4_14_4"])
def test_host_assembly_bitwise_reference(name):
    g = np.load(os.path.join(GOLD, name + ".npz"))
    spec = str(g["spec"])
    parts = spec.split(":")
    prob = pb.make_problem(int(parts[1]), int(parts[2])) if parts[0] == "ex" else pb.baseline_problem(int(parts[1]), int(parts[2]))
    dim = int(g["dim"])
    mesh = pb.MeshConfig.create(dim, list(g["fine"]), list(g["coarse"]), int(g["time_axis"]))
    assert np.array_equal(prob.assemble_rhs(mesh, pb.MeshKind.fine(dim)), g["b_fine"])
    for a in range(dim):
        assert np.array_equal(prob.assemble_rhs(mesh, pb.MeshKind.coarse_along(dim, a)), g[f"b_slab{a}"])
    assert np.array_equal(prob.assemble_rhs(mesh, pb.MeshKind.coarse(dim)), g["b_coarse"])
    if g["exact"].size:
        assert np.array_equal(prob.sample_exact(mesh), g["exact"])


def test_mesh_validation_mirrors_reference():
    with pytest.raises(pb.DivisibilityError):
        pb.MeshConfig.create(2, [10, 10], [4, 4])
    with pytest.raises(pb.DegenerateError):
        pb.MeshConfig.create(2, [4, 4], [4, 4])
    with pytest.raises(pb.DimensionMismatch):
        pb.MeshConfig.create(4, [8] * 4, [2] * 4)
    m = pb.MeshConfig.create(2, [24, 24], [4, 4])
    assert m.factors == [5, 5] and m.point_count(pb.MeshKind.holes_of(2)) == 25 * 16
    assert pb.MeshConfig.create(2, [8, 8], [2, 2]).point_count(pb.MeshKind.holes_of(2)) == 36
    with pytest.raises(pb.UnknownExample):
        pb.make_problem(5, 1)
    # the C-ABI validates the mesh before touching the device
    lib = pb.load_library()
    h = ctypes.c_void_p()
    rc = lib.asdsm_plan_create(2, pb.asdsm._i32([10, 10]), pb.asdsm._i32([4, 4]), -1, pb.asdsm._d3([1, 1, 1]),
                               pb.asdsm._d3([0, 0, 0]), ctypes.byref(h))
    assert rc == 2 and b"not divisible" in lib.asdsm_last_error()


def test_baseline_meshes():
    want = {0: (2, 129, 10), 1: (2, 1029, 20), 2: (2, 4099, 20), 3: (3, 259, 10), 4: (3, 509, 10)}
    for cid, (dim, nf, it) in want.items():
        mesh, iters = pb.baseline_mesh(cid)
        assert mesh.dim == dim and mesh.fine_counts == [nf] * dim and mesh.coarse_counts == [9] * dim and iters == it
    assert pb.baseline_mesh(4)[0].time_axis == 2


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    mesh, _ = pb.baseline_mesh(0)
    with pytest.raises(pb.asdsm.CudaFailure):
        pb.SolverContext(mesh, pb.baseline_problem(0, 0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    q.put((rank, bench.max_over_ranks(1.5 + rank, "cpu")))
    dist.destroy_process_group()


def test_bench_max_over_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: 2.5, 1: 2.5}


def test_cxx_dropin_header_builds_and_fails_loudly_without_gpu(tmp_path):
    """include/asdsm_b200.hpp (the reference's asdsm::asdsm_iterate / SolverContext / errors
    mirrored over the C-ABI) compiles with plain g++, links the in-tree library, and without a GPU
    the solve throws the CudaFailure class -- no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by tests/test_gpu_runner.py")
    from cxx_tools import build_example, run_example
    exe = build_example(tmp_path)
    rc, out = run_example(exe, 1, 1, 99, 9, 3)
    assert rc == 3 and out.startswith("error,CudaFailure"), out


def test_reference_binding_has_no_cpu_fallback():
    """The compiled reference-side binding (tests/cxx/ref_binding.cpp) raises the reference's
    asdsm::Error from the C-ABI status when no GPU is present -- after the reference itself ran."""
    import os
    import subprocess
    import tempfile
    import torch
    binp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "ref_binding")
    if not os.path.exists(binp) or torch.cuda.is_available():
        pytest.skip("needs the built binding and no GPU")
    with tempfile.TemporaryDirectory() as d:
        p = subprocess.run([binp, "ex:1:1", "49", "4", "2", "0", os.path.join(d, "o")], capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 3 and "no CUDA device" in p.stderr
        assert os.path.exists(os.path.join(d, "o.ref.hist.txt"))
