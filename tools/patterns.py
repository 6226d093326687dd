"""Latency-optimal and memory-optimal patterns on a measured B200 profile
(paper Table 4 / PAPER.md:580-602, 617, 647-648).

For a config: measure the cost model (profile_ops), sweep alpha (the
reference's `hetsched sweep` frontier, cli.py:259-306), pick the memory-optimal
alpha for several SLOs (all-GPU latency x {1, 1.5, 3}), execute every chosen
plan for real (execute) and report modelled vs measured latency and the Eq. 4
GPU memory.  usage: python tools/patterns.py [config] [out.json]
"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
out = sys.argv[2] if len(sys.argv) > 2 else None
spec = hs.CONFIGS[cfg]
if cfg == "c2":
    spec = spec.with_(seq=32)  # keep host cells (ms each at H=1024) affordable
w = hs.init_weights(spec)
x = hs.make_input(spec)
ex = hs.RNNExecutor(spec, w)
g = hs.gen_lstm_grid(spec.layers, spec.seq) if spec.dirs == 1 else hs.gen_bilstm_grid(spec.layers, spec.seq)
t0 = time.perf_counter()
cm = hs.profile_ops(g, ex, k=4, reps=5)
prof_s = time.perf_counter() - t0
gpu_plan, cpu_plan = hs.baseline_plans(g, cm)
gpu_lat = hs.evaluate(g, cm, gpu_plan).latency


def measure(plan, reps=5):
    hs.execute(g, plan, ex, x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        hs.execute(g, plan, ex, x)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return statistics.median(ts)


rows = []
for name, plan in [("gpu", gpu_plan), ("cpu", cpu_plan), ("latency-optimal", hs.latency_optimal_plan(g, cm))]:
    ev = hs.evaluate(g, cm, plan)
    rows.append({"pattern": name, "alpha": plan.alpha, "k_star": plan.k_star,
                 "gpu_nodes": sum(1 for s in plan.selection if s == 0), "model_latency_ms": ev.latency,
                 "gpu_memory_mb": ev.gpu_memory, "measured_wall_ms": measure(plan, 3 if name == "cpu" else 5)})
for slo_x in (1.0, 1.5, 3.0):
    pt = hs.memory_optimal_alpha(g, cm, slo_ms=gpu_lat * slo_x, alphas="0:2:0.1")
    rows.append({"pattern": f"memory-optimal (SLO = {slo_x} x GPU)", "alpha": pt.alpha, "k_star": pt.k_star,
                 "gpu_nodes": sum(1 for s in pt.plan.selection if s == 0), "model_latency_ms": pt.latency,
                 "gpu_memory_mb": pt.gpu_memory, "measured_wall_ms": measure(pt.plan)})
res = {"config": cfg, "spec": str(spec), "n_nodes": g.n, "profile_seconds": prof_s,
       "W_gpu_ms_per_cell": float(cm.W[:, 0].mean()), "W_host_ms_per_cell": [float(v) for v in cm.W[0, 1:]],
       "b_MB_per_ms": cm.b, "rows": rows}
print(json.dumps(res, indent=1))
if out:
    Path(out).write_text(json.dumps(res, indent=1) + "\n")
