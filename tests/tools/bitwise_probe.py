"""Probe: which solves are bitwise equal between batched (batch-minor) and single-signal runs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1604_06236_b200 as nf
from oracle import nfft_oracle as O

for logP in [int(a) for a in sys.argv[1:]] or [12, 16, 18]:
    P, B = 1 << logP, 16
    t, data = O.make_inputs(P, 0.3, B, 16046)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    out = []
    for name, fn in (("type5", nf.type5), ("type4", nf.type4)):
        full = fn(plan, data); one = fn(plan, data[B - 1])
        out.append(f"{name} {np.array_equal(full[B-1], one)} {O.rel_l2(one, full[B-1]):.1e}")
    for name, fn in (("r5", nf.refine_type5), ("r4", nf.refine_type4)):
        full = fn(plan, data, passes=1); one = fn(plan, data[B - 1], passes=1)
        out.append(f"{name} {np.array_equal(full[B-1], one)} {O.rel_l2(one, full[B-1]):.1e}")
    print(f"P=2^{logP}:", " | ".join(out))
