"""Command-line driver mirroring the reference's `asdsm` CLI (proj/src/cli.cpp:86-155):

  python -m paper_2303_01163_b200.cli run      [--example E --setting S --nf N --nc C --tol T
                                                --max-iter K --seed S --subsample F --out PATH
                                                --config FILE]
  python -m paper_2303_01163_b200.cli snapshot [same flags] [--at-iter K]

Exit codes as the reference: 0 ok, 2 usage/configuration error, 3 singular operator.
(`verify` suites are the reference's self-test harness; see tests/ for ours.)
"""
import argparse
import sys

from . import asdsm as A

KEYS = {"example": int, "setting": int, "nf": int, "nc": int, "tol": float, "max-iter": int, "seed": int,
        "subsample": float, "out": str, "at-iter": int}


def _apply_config_file(path, cfg, extra):
    """apply_config_file (cli.cpp:46-76): key=value lines, '#' comments; flags override."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise A.Error(f"config: cannot read {path}")
    for lineno, line in enumerate(lines, 1):
        text = line.strip()
        if not text or text.startswith("#"):
            continue
        if "=" not in text:
            raise A.Error(f"config: expected key=value at line {lineno}")
        key, value = (x.strip() for x in text.split("=", 1))
        if key not in KEYS:
            raise A.Error(f"config: unknown key '{key}'")
        try:
            v = KEYS[key](value)
        except ValueError:
            raise A.Error(f"config: bad value for '{key}' at line {lineno}")
        if key == "at-iter":
            extra["at_iter"] = v
        else:
            setattr(cfg, key.replace("-", "_"), v)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser(prog="asdsm")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "snapshot"):
        p = sub.add_parser(name)
        for k, t in KEYS.items():
            if k == "at-iter" and name == "run":
                continue
            p.add_argument("--" + k, type=t, default=None)
        p.add_argument("--config", default=None)
    try:
        ns = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    cfg = A.RunConfig()
    extra = {"at_iter": 20}
    try:
        if ns.config:
            _apply_config_file(ns.config, cfg, extra)
        for k in KEYS:
            v = getattr(ns, k.replace("-", "_"), None)
            if v is None:
                continue
            if k == "at-iter":
                extra["at_iter"] = v
            else:
                setattr(cfg, k.replace("-", "_"), v)
        if ns.cmd == "run":
            res = A.run_experiment(cfg)
            if cfg.out:
                print(f"wrote {cfg.out}: {len(res.state.history)} rows, stopped by {res.state.stop_reason}")
            else:
                sys.stdout.write(res.csv)
            return 0
        grid = A.residual_snapshot(cfg, extra["at_iter"])
        if cfg.out:
            A.write_text_file(cfg.out, grid)
            print(f"wrote {cfg.out}")
        else:
            sys.stdout.write(grid)
        return 0
    except A.SingularMatrix as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return 3
    except Exception as e:  # noqa: BLE001 - mirror the reference's catch-all -> exit 2
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
