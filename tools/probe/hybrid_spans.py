"""Per-span breakdown of one hybrid plan execution (c1, half the steps on the
host): node spans, transfers and the makespan, to locate the executor's fixed
costs the cost model has no term for."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402
from paper_2307_11339_b200.planner import Plan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
first = len(sys.argv) > 2 and sys.argv[2] == "first"
spec = hs.CONFIGS[cfg]
ex = hs.RNNExecutor(spec, hs.init_weights(spec))
x = hs.make_input(spec)
g = hs.gen_lstm_grid(spec.layers, spec.seq)
cm = hs.profile_ops(g, ex, k=4, reps=5)
lat = hs.latency_optimal_plan(g, cm)
T = spec.seq
sel = [1 if ((v % T < T // 2) if first else (v % T >= T // 2)) else 0 for v in range(g.n)]
cores, _a, _l = hs.resolve_cores(g, cm, lat.order.seq, sel, 1)
plan = Plan(order=lat.order, selection=tuple(sel), cores=tuple(cores), k_star=1, alpha=0.0)
print("modelled", hs.evaluate(g, cm, plan).latency)
for _ in range(3):
    hs.execute(g, plan, ex, x)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    r = hs.execute(g, plan, ex, x)
    torch.cuda.synchronize()
    print("wall ms", (time.perf_counter() - t0) * 1e3, "makespan", r.trace.makespan)
for sp in r.trace.nodes:
    print(f"node {sp.node:3d} dev {sp.device} {sp.start:8.3f} {sp.end:8.3f} {sp.end - sp.start:7.3f}")
for tr in r.trace.transfers:
    print(f"xfer {tr.src:3d}->{tr.dst:3d} {tr.start:8.3f} {tr.end:8.3f}")
