"""Back-to-back device solves of quadrotor N=1e5 with per-phase timings (OCG_TIMING=1):
the plan-time variance evidence in profiles/r1_v14_plan_spikes_*.txt."""
import sys, time
sys.path.insert(0, '.')
from paper_2510_03932_b200 import MODELS, Model, solve
m = Model(MODELS["quadrotor"], 100000)
solve(m, max_iter=1)
for i in range(10):
    print("=== solve", i, file=sys.stderr, flush=True)
    t = time.perf_counter(); r = solve(m)
    print("wall", round(time.perf_counter() - t, 3), round(r["time_total"], 3), round(r["time_plan_eval"], 3), round(r["time_plan_kkt"], 3), round(r["time_plan_ldl"], 3), round(r["time_setup"], 3), file=sys.stderr, flush=True)
