"""Repeat the 40^3 first Newton pass from the same state and check that every repetition gives the
same counts, histories and solution bit for bit (the dataflow sweeps spin on tagged words: any
ordering bug would show up as run-to-run differences or a trapped wait).

    python scripts/stress_determinism.py [N] [REPS]
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cp = CubeProblem(n=n, nu=0.5)
ctx = cp.context(0)
ctx.set_state(cp.seeded_state())
ctx.state_save()
opts = cp.solver_options()
ref = None
bad = 0
for r in range(reps):
    ctx.state_restore()
    out = ctx.newton_first_pass(cp.ts, opts)
    key = (hashlib.sha256(np.ascontiguousarray(out["x"]).tobytes()).hexdigest(),
           hashlib.sha256(np.ascontiguousarray(out["history"]).tobytes()).hexdigest(),
           tuple(sorted((k, int(v)) for k, v in out["stats"].items() if k != "t_solve")))
    if ref is None:
        ref = key
    elif key != ref:
        bad += 1
        print("repetition", r, "differs", flush=True)
print(json.dumps(dict(n=n, reps=reps, differing=bad, x_sha256=ref[0][:16], stats=dict(ref[2]))), flush=True)
sys.exit(1 if bad else 0)
