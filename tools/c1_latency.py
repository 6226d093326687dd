"""c1 (reference toy DAG, latency-optimal partition): measured profile ->
latency-optimal plan -> execute; p50 latency of the fused forward, the plan
execution and CPU fused torch for context."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

spec = hs.CONFIGS["c1"]
w = hs.init_weights(spec)
x = hs.make_input(spec)
ex = hs.RNNExecutor(spec, w)
g = hs.gen_lstm_grid(spec.layers, spec.seq)
cm = hs.profile_ops(g, ex, k=4, reps=20)
plan = hs.latency_optimal_plan(g, cm)
ev = hs.evaluate(g, cm, plan)
mem = hs.memory_optimal_alpha(g, cm)
xd = x.cuda()
outs = ex.alloc_outputs()


def p50(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
dev_ms = []
for _ in range(200):
    e0.record()
    ex.forward(xd, out=outs)
    e1.record()
    e1.synchronize()
    dev_ms.append(e0.elapsed_time(e1))
m = torch.nn.LSTM(spec.I, spec.hidden, spec.layers)
with torch.no_grad():
    cpu = p50(lambda: m(x), 100)
res = {
    "config": "c1", "plan_gpu_nodes": sum(1 for s_ in plan.selection if s_ == 0), "plan_k_star": plan.k_star,
    "plan_model_latency_ms": ev.latency, "memory_optimal_alpha": mem.alpha,
    "fused_forward_device_p50_ms": statistics.median(dev_ms),
    "fused_forward_wall_p50_ms": p50(lambda: ex.forward(xd, out=outs)),
    "execute_plan_wall_p50_ms": p50(lambda: hs.execute(g, plan, ex, x), 50),
    "cpu_torch_fused_p50_ms": cpu, "cpu_threads": torch.get_num_threads(),
    "profile_W_gpu_ms_per_cell": float(cm.W[0, 0]), "profile_W_host_ms_per_cell_1core": float(cm.W[0, 1]),
    "link_MB_per_ms": cm.b,
}
print(json.dumps(res))
