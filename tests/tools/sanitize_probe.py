#!/usr/bin/env python
"""Small end-to-end exercise of every kernel family for compute-sanitizer runs:
plans (eta 2, 3, 1.5), refined solves single / batched (signal-major and
batch-minor chains), forward NFFTs, generic sizes, clustered nodes."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1604_06236_b200 as nf
from oracle import nfft_oracle as O

for P, B, J, eta in ((64, 1, 0.3, 2), (1024, 20, 0.3, 2), (1024, 3, 0.45, 3), (4096, 1, 0.3, 1.5), (1000, 4, 0.3, 2),
                     (4096, 40, 0.3, 2)):
    t, data = O.make_inputs(P, J, B, 5)
    g = nf.validate_grid(t)
    prm = nf.MethodParams.from_mu(1e-15, P, eta, fractional_eta=float(eta) != int(eta))
    plan = nf.build_plan(g, prm)
    x = data if B > 1 else data[0]
    r5 = nf.refine_type5(plan, x, passes=1)
    r4 = nf.refine_type4(plan, x, passes=1)
    a = nf.nfft_type1(g, x, P)
    s = nf.nfft_type2(x, g)
    print(P, B, eta, float(np.abs(r5).max()), float(np.abs(r4).max()), float(np.abs(a).max()), float(np.abs(s).max()),
          flush=True)
# clustered nodes: persistent-gather fallback blocks
P, B = 4096, 40
sp = np.ones(P); sp[1000:1064] = 1.7; sp *= P / sp.sum()
t = (np.cumsum(sp) - sp[0] * 0.5) / P
plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
x = (np.random.default_rng(3).standard_normal((B, P)) + 1j) / 2
print("clustered", float(np.abs(nf.refine_type4(plan, x, passes=1)).max()), flush=True)
print("OK")
