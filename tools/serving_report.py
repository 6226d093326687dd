"""Table-6-style serving study on one B200 with measured inputs (SURVEY §8f
row 3, servingsim.py:143-288).

The nine models are the paper's nine feasible structures (Table 4,
:580-602): LSTM <layers, batch, io, seq> = the baseline <12, 8, 64, 96> and
its one-parameter variants layers 8/16, batch 1/2/4, io 32, seq 32/64.

1. Each model runs on the B200 executor; ResidencyServer measures its HBM
   footprint (packed weights + workspace + request staging), the packed
   weight bytes a swap moves, the warm request latency (host buffers in and
   out, CUDA events) and the H2D load bandwidth.
2. The Chrion loop per model (profile_ops -> latency-optimal plan ->
   memory-optimal alpha under SLO = the all-GPU latency) gives the
   latency-optimal and memory-optimal variants: latency = the plan executed
   for real (execute, wall clock), footprint = the measured all-GPU footprint
   scaled by the plan's Eq. 4 GPU memory over the all-GPU plan's.
3. Serving, uniform requests over the nine models, HBM budget = a fraction of
   the summed footprints so the resident set cannot hold every model:
   * REAL: ResidencyServer.serve (evictions free device memory, loads upload
     the packed weights, every request runs the forward);
   * SIMULATED: run_serving over the measured scalars (the reference's
     accounting) — swaps must agree exactly, violations closely;
   * PATTERNS: compare_patterns over the three variants (Table 6).

usage: python tools/serving_report.py [out.json] [--requests N] [--capacity-frac F]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402
from paper_2307_11339_b200.serving import ModelEntry, ResidencyServer, Workload, compare_patterns, run_serving  # noqa: E402

# <layers, batch, io, seq>: baseline and its feasible variants
NINE = {"base": (12, 8, 64, 96), "L8": (8, 8, 64, 96), "L16": (16, 8, 64, 96), "B1": (12, 1, 64, 96),
        "B2": (12, 2, 64, 96), "B4": (12, 4, 64, 96), "IO32": (12, 8, 32, 96), "S32": (12, 8, 64, 32),
        "S64": (12, 8, 64, 64)}


def wall(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?")
    ap.add_argument("--requests", type=int, default=180)
    ap.add_argument("--capacity-frac", type=float, default=0.6)
    ap.add_argument("--no-patterns", action="store_true")
    args = ap.parse_args()

    models, specs = {}, {}
    for i, (k, (L, B, io, T)) in enumerate(NINE.items()):
        specs[k] = hs.RNNSpec("lstm", L, io, T, B, input=io)
        models[k] = hs.RNNExecutor(specs[k], hs.init_weights(specs[k], i))
    probe = ResidencyServer(models, capacity_mb=1e12)
    gpu_ms = {k: probe.warm_latency(k, reps=9) for k in models}
    bw = probe.load_bandwidth_mb_per_ms(max(models, key=lambda k: probe.weights_mb[k]))
    gpu_entries = probe.entries(gpu_ms)

    per_model = {}
    lat_entries, mem_entries = [], []
    for e in gpu_entries:
        k, spec, ex = e.id, specs[e.id], models[e.id]
        row = {"shape": dict(zip(("layers", "batch", "io", "seq"), NINE[k])), "plan": ex.plan(),
               "footprint_mb": e.gpu_footprint_mb, "weights_mb": e.weights_mb, "gpu_request_ms": e.exec_latency_ms,
               "slo_ms": e.slo_ms}
        if not args.no_patterns:
            ex.load()  # the probe's measurements leave models offloaded
            g = hs.gen_lstm_grid(spec.layers, spec.seq)
            x = hs.make_input(spec)
            cm = hs.profile_ops(g, ex, k=4, reps=3)
            gpu_plan, _ = hs.baseline_plans(g, cm)
            ev_gpu = hs.evaluate(g, cm, gpu_plan)
            lo = hs.latency_optimal_plan(g, cm)
            mo = hs.memory_optimal_alpha(g, cm, slo_ms=ev_gpu.latency, alphas="0:2:0.1")
            for name, plan, dst in (("latency-optimal", lo, lat_entries), ("memory-optimal", mo.plan, mem_entries)):
                ev = hs.evaluate(g, cm, plan)
                frac = ev.gpu_memory / ev_gpu.gpu_memory if ev_gpu.gpu_memory > 0 else 1.0
                gpu_cells = sum(1 for s in plan.selection if s == 0)
                if gpu_cells == g.n:
                    ms = e.exec_latency_ms  # the all-GPU plan runs the fused request path
                else:
                    ms = wall(lambda: hs.execute(g, plan, ex, x), 3)
                dst.append(ModelEntry(k, e.gpu_footprint_mb * frac, ms, e.weights_mb * frac, e.slo_ms))
                row[name] = {"alpha": plan.alpha, "gpu_cells": gpu_cells, "cells": g.n, "memory_frac": frac,
                             "model_latency_ms": ev.latency, "latency_ms": ms}
            row["W_gpu_ms_per_cell"] = float(cm.W[:, 0].mean())
            row["W_host_ms_per_cell"] = float(cm.W[:, 1].mean())
        per_model[k] = row
        print(k, json.dumps(row), flush=True)

    total = sum(e.gpu_footprint_mb for e in gpu_entries)
    cap = max(args.capacity_frac * total, max(e.gpu_footprint_mb for e in gpu_entries) * 1.001)
    w = Workload(args.requests, "uniform")
    srv = ResidencyServer(models, capacity_mb=cap, slo_ms={e.id: e.slo_ms for e in gpu_entries})
    real, meas = srv.serve(w)
    sim = run_serving(gpu_entries, cap, w, bw)
    res = {
        "device": torch.cuda.get_device_name(), "models": per_model, "capacity_mb": cap, "total_footprint_mb": total,
        "load_bandwidth_mb_per_ms": bw, "workload": {"requests": args.requests, "pattern": "uniform"},
        "real": {"slo_violation": real.metrics.slo_violation, "swapping_rate": real.metrics.swapping_rate,
                 "swaps": real.metrics.swaps, "violations": real.metrics.violations,
                 "p50_latency_ms": statistics.median(m.latency_ms for m in meas),
                 "p50_load_ms": statistics.median([m.load_ms for m in meas if m.load_ms > 0] or [0.0]),
                 "p50_evict_ms": statistics.median([m.evict_ms for m in meas if m.evict_ms > 0] or [0.0]),
                 "p50_exec_ms": statistics.median(m.exec_ms for m in meas)},
        "simulated_on_measured_scalars": {"slo_violation": sim.metrics.slo_violation,
                                          "swapping_rate": sim.metrics.swapping_rate, "swaps": sim.metrics.swaps,
                                          "violations": sim.metrics.violations},
    }
    if not args.no_patterns:
        rep = compare_patterns(gpu_entries, lat_entries, mem_entries, cap, w, bw)
        res["patterns_table6"] = rep.metrics()
    print(json.dumps(res, indent=1))
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
