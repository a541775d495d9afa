"""Golden rows of the reference's Monte-Carlo harness (build container only).

Run:  python oracle/make_sweep_golden.py [/root/reference]

Imports the reference package ``nufft1d`` from ``<ref>/pkg/src`` (read-only),
runs its ``run_sweep`` / ``run_figure`` (bench.py:128-206, 268-301) on small
seeded configurations and writes ``tests/golden/sweep_rows.json``.  The GPU
harness (paper_1604_06236_b200/bench.py) is compared with these rows in
tests/test_gpu_cli_bench.py: same row keys in the same order, equal
data-independent flop totals, CG iteration counts within one, and errors at
the reference's own level.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)

CASES = {
    # name: (kind, kwargs) — small enough for the CPU reference in seconds
    "sweep_all": ("sweep", dict(p=(16, 64), eta=(1, 2), mu=(1e-15, 1e-10, 1e-6), trials=3, seed=5)),
    "sweep_passes2": ("sweep", dict(p=(32,), eta=(1, 3), mu=(1e-18, 1e-12, 1e-8), trials=2, seed=11,
                                    methods=("NFFT", "R-NFFT"), refine_passes=2)),
    "fig2": ("figure", dict(p=(32, 64), eta=(1, 2), mu=(1e-14, 1e-10, 1e-6), trials=2, seed=3)),
    "fig6": ("figure", dict(p=(16, 32), trials=2, seed=7)),
}


def main(ref_root="/root/reference"):
    sys.path.insert(0, os.path.join(ref_root, "pkg", "src"))
    import nufft1d.bench as RB  # the reference harness

    out = {}
    for name, (kind, kw) in CASES.items():
        if kind == "sweep":
            cfg = RB.TrialConfig(**kw)
            rows = RB.run_sweep(cfg)
            meta = None
        else:
            fig = name
            cfg = dataclasses.replace(RB.FIGURE_DEFAULTS[fig], **kw)
            rows, meta = RB.run_figure(fig, cfg)
        out[name] = {"kind": kind, "config": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                     "meta": meta, "rows": [dataclasses.asdict(r) for r in rows]}
        print(name, len(rows), "rows")
    # the trial streams themselves (reference generate_trial, bench.py:84-92)
    out["trial_streams"] = []
    for P, seed in ((16, 0), (16, 5 ^ 2), (64, 11), (1024, 3)):
        grid, amp = RB.generate_trial(P, seed)
        out["trial_streams"].append({"P": P, "seed": seed, "nodes": [float(v) for v in grid.instants],
                                     "re": [float(v) for v in amp.real], "im": [float(v) for v in amp.imag]})
    path = os.path.join(REPO, "tests", "golden", "sweep_rows.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path)


if __name__ == "__main__":
    main(*sys.argv[1:])
