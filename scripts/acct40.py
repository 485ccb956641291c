"""Per kernel@level device time of the 40^3 first pass (live accounting), for sweep tuning."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem
n = int(os.environ.get("N", "40"))
cp = CubeProblem(n=n, nu=0.5, dt=float(os.environ.get("DT", "1e-3")))
ctx = cp.context(0)
st = cp.seeded_state()
ctx.set_state(st)
ctx.state_save()
opts = cp.solver_options()
for _ in range(int(os.environ.get("WARM", "2"))):
    ctx.state_restore()
    out = ctx.newton_first_pass(cp.ts, opts)
ctx.kernel_accounting(True)
ctx.state_restore()
ctx.timer_start()
out = ctx.newton_first_pass(cp.ts, opts)
ms = ctx.timer_stop()
acc = ctx.kernel_account()
ctx.kernel_accounting(False)
tag = os.environ.get("TAG", "")
print(f"== {tag} pass {ms:.1f} ms  fgmres {out['times']['fgmres_ms']:.1f}  setup {out['times']['amg_setup_ms']:.1f} host {out['times']['amg_host_ms']:.1f}")
for k, (nl, t, by) in sorted(acc.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"   {k:28s} launches {nl:5d}  {t:8.2f} ms  {t / max(nl, 1) * 1e3:8.1f} us/launch")
