#!/usr/bin/env python
"""A/B bitwise check of the small-batch gridding kernels against the legacy
ones: `python scripts/small_ab.py save DIR` under each setting
(NFFT45_LEGACY_SMALL=1 or not), then `python scripts/small_ab.py cmp A B`."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CASES = [(8, 1, 0.3), (32, 1, 0.0), (64, 1, 0.3), (64, 3, 0.45), (1000, 2, 0.3), (4096, 5, 0.3),
         (4096, 1, 0.1), (1 << 16, 1, 0.3), (1 << 16, 7, 0.45), (1 << 20, 1, 0.4), (3 * 1024, 4, 0.3)]


def run(outdir):
    import paper_1604_06236_b200 as nf
    os.makedirs(outdir, exist_ok=True)
    for P, B, J in CASES:
        rng = np.random.default_rng(P + B)
        t = np.sort(((np.arange(P) + rng.uniform(-J, J, P)) / P) % 1.0)
        if J == 0.0:
            t = np.arange(P) / P
        perm = rng.permutation(P)
        grid = nf.validate_grid(t[perm])
        a = (rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))) / np.sqrt(2)
        A1 = nf.nfft_type1(grid, a if B > 1 else a[0], P)
        A2 = nf.nfft_type2(a if B > 1 else a[0], grid)
        np.save(f"{outdir}/t1_{P}_{B}.npy", A1)
        np.save(f"{outdir}/t2_{P}_{B}.npy", A2)
        if P in (64, 4096, 1 << 16, 1 << 20):
            params = nf.MethodParams.from_mu(1e-15, P, 2)
            plan = nf.build_plan(grid, params)
            np.save(f"{outdir}/r5_{P}_{B}.npy", nf.refine_type5(plan, a if B > 1 else a[0], passes=1))
            np.save(f"{outdir}/r4_{P}_{B}.npy", nf.refine_type4(plan, a if B > 1 else a[0], passes=1))
            np.save(f"{outdir}/ks_{P}_{B}.npy", plan.kernel_data.kernel_samples)
    print("saved", outdir)


def cmp(da, db):
    bad = 0
    for f in sorted(os.listdir(da)):
        x, y = np.load(f"{da}/{f}"), np.load(f"{db}/{f}")
        same = np.array_equal(x.view(np.uint64), y.view(np.uint64))
        rel = np.linalg.norm(x - y) / max(np.linalg.norm(x), 1e-300)
        print(f"{f:24s} {'bitwise' if same else 'DIFF'} rel={rel:.2e}")
        bad += not same
    print("ALL BITWISE" if not bad else f"{bad} differ")


if __name__ == "__main__":
    if sys.argv[1] == "save":
        run(sys.argv[2])
    else:
        cmp(sys.argv[2], sys.argv[3])
