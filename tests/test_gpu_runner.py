"""GPU: the runner layer (runner.hpp) and the stop rules against the reference."""
import os

import numpy as np
import pytest

import paper_2303_01163_b200 as pb
from ref_tools import eval_floor, have_ref, ref_bundle, ref_iterate

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("ex,st,nf,nc", [(1, 1, 99, 9), (3, 1, 99, 9), (1, 1, 24, 4)])
def test_run_experiment_default_options_match_reference(ex, st, nf, nc, tmp_path):
    """Default IterateOptions (tol 1e-12, stagnation window 3 / ratio 0.99): same number of
    rows, same stop reason, same residual history (floor-aware) as the reference."""
    out = tmp_path / "h.csv"
    res = pb.run_experiment(pb.RunConfig(example=ex, setting=st, nf=nf, nc=nc, out=str(out)))
    ref = ref_iterate(f"ex:{ex}:{st}", nf, nc, 20, 0, env={"REF_DUMP_DEFAULT_OPTS": "1"})
    assert res.state.stop_reason == ref["stop"]
    assert len(res.state.history) == len(ref["hist"])
    got = np.array([h.res_l2 for h in res.state.history])
    want = ref["hist"][:, 1]
    floor = eval_floor(ref_bundle(f"ex:{ex}:{st}", nf, nc), ref["u"])  # fp64 floor of b - Au
    assert np.all(np.abs(got - want) <= np.maximum(1e-8 * want, floor))
    text = out.read_text().splitlines()
    assert text[0] == "k,res_l2,res_inf,err_max,err_l2,s_hat,wall_ms"
    assert len(text) == 1 + len(res.state.history)
    row0 = text[1].split(",")
    assert row0[0] == "0" and row0[5] == "nan" and float(row0[6]) >= 0.0
    assert all(h.wall_ms >= 0.0 for h in res.state.history)


def test_residual_snapshot_matches_reference():
    cfg = pb.RunConfig(example=2, setting=1, nf=99, nc=9, max_iter=20)
    grid = pb.residual_snapshot(cfg, 5)
    rows = [list(map(float, line.split(","))) for line in grid.strip().splitlines()]
    assert len(rows) == 99 and all(len(r) == 99 for r in rows)
    ref = ref_iterate("ex:2:1", 99, 9, 5, 0)
    r = np.abs(ref["r"]).reshape(99, 99)
    scale = np.max(r)
    assert np.max(np.abs(np.array(rows) - r)) <= 1e-6 * scale


def test_cli_run_and_errors(tmp_path, capsys):
    from paper_2303_01163_b200 import cli
    assert cli.main(["run", "--nf", "10", "--nc", "4"]) == 2  # divisibility -> exit 2
    cfgf = tmp_path / "c.cfg"
    cfgf.write_text("# comment\nexample=1\nnf=24\nnc=4\nmax-iter=3\n")
    assert cli.main(["run", "--config", str(cfgf), "--seed", "1"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0].startswith("k,res_l2") and len(out) == 1 + 4
