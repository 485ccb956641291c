"""Time setup phases and one Newton first pass at a given cube size on cuda:0."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1809_06350_b200 import CubeProblem

for n in [int(a) for a in sys.argv[1:]] or [40]:
    nu = 0.5 if n in (40, 160) else 0.45
    dt = float(os.environ.get("DT", "1e-3"))
    t = time.time(); cp = CubeProblem(n=n, nu=nu, dt=dt); t_mesh = time.time() - t
    t = time.time(); ctx = cp.context(0); t_ctx = time.time() - t
    st = cp.seeded_state()
    ctx.set_state(st)
    opts = cp.solver_options()
    mx = int(os.environ.get("MAXIT", "0"))
    if mx:  # profiling only: cap every Krylov solve
        for c in (opts.outer, opts.a, opts.s, opts.inner):
            c.max_iters = min(c.max_iters, mx)
    for rep in range(int(os.environ.get("REPS", "2"))):
        t = time.time(); out = ctx.newton_first_pass(cp.ts, opts); t_pass = time.time() - t
        ctx.set_state(st)
        print(json.dumps(dict(n=n, nu=nu, rep=rep, mesh_s=round(t_mesh, 2), ctx_s=round(t_ctx, 2), pass_s=round(t_pass, 3),
                              norm=out["norm"], stats=out["stats"], hist=list(out["history"]), times=out["times"])), flush=True)
