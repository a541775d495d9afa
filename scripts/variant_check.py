"""Bitwise check of an env-switch kernel variant against the default build on batch-minor
chain shapes: python scripts/variant_check.py NFFT45_HYB=0 [more VAR=VAL ...]"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[2])
import paper_1604_06236_b200 as nf
out = {}
for P, B, J in [(4096, 32, 0.3), (1 << 16, 16, 0.3), (1 << 16, 300, 0.3), (1 << 15, 24, 0.3), (1 << 17, 40, 0.3), (12288, 16, 0.3)]:
    rng = np.random.default_rng(P + B)
    t = np.mod((np.arange(P) + rng.uniform(-J, J, P)) / P, 1.0)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    x = (rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))) / np.sqrt(2)
    out[f"t5_{P}_{B}"] = nf.refine_type5(plan, x, passes=1)
    out[f"t4_{P}_{B}"] = nf.refine_type4(plan, x, passes=2)
np.savez(sys.argv[1], **out)
"""

if __name__ == "__main__":
    extra = dict(a.split("=", 1) for a in sys.argv[1:])
    outs = []
    with tempfile.TemporaryDirectory() as d:
        for i, env in enumerate(({}, extra)):
            f = os.path.join(d, f"v{i}.npz")
            subprocess.run([sys.executable, "-c", SCRIPT, f, ROOT], check=True, env=dict(os.environ, **env), timeout=600)
            outs.append(dict(np.load(f)))
    bad = [k for k in outs[0] if not np.array_equal(outs[0][k], outs[1][k])]
    for k in outs[0]:
        print(k, "bitwise" if k not in bad else "DIFF %.3e" % (np.linalg.norm(outs[0][k] - outs[1][k]) / np.linalg.norm(outs[0][k])))
    sys.exit(1 if bad else 0)
