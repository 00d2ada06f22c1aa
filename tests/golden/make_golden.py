"""Regenerate tests/golden/*.npz from the reference's own code (oracle/_ref/ref_dump).

Run here (needs oracle/_ref built from /root/reference):  python tests/golden/make_golden.py
Each fixture holds the reference's residual history, initial guess, final iterate and
residual, plus the history of the same run under a different (equally valid) fill ordering
of its direct solver (`hist_cm`), which measures the reference's own reproducibility floor.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from ref_tools import ref_bundle, ref_iterate  # noqa: E402

CASES = [
    # name, spec, nf, nc, iters, seed
    ("ex1s1_24_4", "ex:1:1", 24, 4, 10, 0),
    ("ex1s1_49_4", "ex:1:1", 49, 4, 12, 3),
    ("ex3s1_24_4", "ex:3:1", 24, 4, 10, 1),
    ("ex4s1_14_4", "ex:4:1", 14, 4, 5, 0),
    ("cfg0_39_9", "cfg:0:0", 39, 9, 10, 0),
    ("cfg1_49_4", "cfg:1:7", 49, 4, 12, 2),
    ("cfg2_49_4", "cfg:2:5", 49, 4, 12, 0),
    ("cfg3_14_4", "cfg:3:0", 14, 4, 5, 1),
    ("cfg4_14_4", "cfg:4:3", 14, 4, 5, 2),
]

if __name__ == "__main__":
    for name, spec, nf, nc, it, seed in CASES:
        ref = ref_iterate(spec, nf, nc, it, seed)
        alt = ref_iterate(spec, nf, nc, it, seed, env={"ASDSM_STUB_ORDER": "cm"})
        bun = ref_bundle(spec, nf, nc)
        dim, ta, fnf, fnc = ref["meta"]
        np.savez_compressed(os.path.join(HERE, name + ".npz"), spec=spec, nf=nf, nc=nc, iters=it, seed=seed,
                            dim=dim, time_axis=ta, fine=np.array(fnf), coarse=np.array(fnc), hist=ref["hist"],
                            hist_cm=alt["hist"], u=ref["u"], r=ref["r"], u0=ref["u0"], b_fine=bun["fine"],
                            b_coarse=bun["coarse"], **{f"b_slab{a}": bun["aniso"][a] for a in range(dim)},
                            exact=bun.get("exact", np.zeros(0)))
        print(name, "k=0..%d" % (len(ref["hist"]) - 1), "res", ref["hist"][0, 1], "->", ref["hist"][-1, 1])
