"""Modelled vs measured latency of hybrid CPU/GPU plans.

For a config: measure the cost model (profile_ops: per-cell GPU times from
hs_rnn_profile_cells, host cells under j-way contention), then for a set of
plans — all-GPU, latency-optimal, memory-optimal at SLO 1.5x and 3x the
all-GPU latency, and forced layer splits (the first / last layer on the
host) — compare the planner's modelled latency (evaluate, engine.py:167-210)
with the measured makespan of executing the plan for real (execute ->
Trace.makespan, the reference's definition: last node end; GPU segments on
the fused forward's kernels).  ``wall_ms`` adds the executor's final output
assembly.

usage: python tools/hybrid_model_check.py [config] [out.json] [--seq T]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402
from paper_2307_11339_b200.planner import Plan  # noqa: E402


def pinned(g, cm, order, sel, k_star):
    """A device-class assignment pinned to concrete cores the way the planner
    pins its own (engine.resolve_cores, engine.py:213-262)."""
    cores, _aft, _lat = hs.resolve_cores(g, cm, order.seq, sel, k_star)
    return Plan(order=order, selection=tuple(sel), cores=tuple(cores), k_star=k_star if any(sel) else 0, alpha=0.0)


def layer_split(g, cm, spec, host_layers, order, k_star=1):
    T, D = spec.seq, spec.dirs
    sel = [1 if (v // T) // D in host_layers else 0 for v in range(g.n)]
    return pinned(g, cm, order, sel, k_star)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c1")
    ap.add_argument("out", nargs="?")
    ap.add_argument("--seq", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    spec = hs.CONFIGS[args.config]
    if args.seq:
        spec = spec.with_(seq=args.seq)
    ex = hs.RNNExecutor(spec, hs.init_weights(spec))
    x = hs.make_input(spec)
    g = hs.gen_lstm_grid(spec.layers, spec.seq) if spec.dirs == 1 else hs.gen_bilstm_grid(spec.layers, spec.seq)
    cm = hs.profile_ops(g, ex, k=4, reps=5)
    gpu_plan, _ = hs.baseline_plans(g, cm)
    gpu_lat = hs.evaluate(g, cm, gpu_plan).latency
    lat_opt = hs.latency_optimal_plan(g, cm)
    plans = [("all-gpu", gpu_plan), ("latency-optimal", lat_opt)]
    for x_slo in (1.5, 3.0):
        pt = hs.memory_optimal_alpha(g, cm, slo_ms=gpu_lat * x_slo, alphas="0:4:0.1")
        plans.append((f"memory-optimal SLO {x_slo}x", pt.plan))
    if spec.layers >= 2:
        plans.append(("layer 0 on host", layer_split(g, cm, spec, {0}, lat_opt.order)))
        plans.append((f"layer {spec.layers - 1} on host", layer_split(g, cm, spec, {spec.layers - 1}, lat_opt.order)))
        plans.append(("layers 0 and 1 on host, 2 cores", layer_split(g, cm, spec, {0, 1}, lat_opt.order, 2)))
    else:
        T = spec.seq
        sel = [1 if v % T >= T // 2 else 0 for v in range(g.n)]
        plans.append(("second half of the steps on host", pinned(g, cm, lat_opt.order, sel, 1)))
        sel = [1 if v % T < T // 2 else 0 for v in range(g.n)]
        plans.append(("first half of the steps on host", pinned(g, cm, lat_opt.order, sel, 1)))
    rows = []
    for name, plan in plans:
        model = hs.evaluate(g, cm, plan).latency
        hs.execute(g, plan, ex, x)
        torch.cuda.synchronize()
        ms, wall = [], []
        for _ in range(args.reps):
            res = hs.execute(g, plan, ex, x)
            torch.cuda.synchronize()
            ms.append(res.trace.makespan)
            wall.append(res.wall_ms)
        meas = statistics.median(ms)
        rows.append({"plan": name, "gpu_cells": sum(1 for s in plan.selection if s == 0), "cells": g.n,
                     "k_star": plan.k_star, "modelled_ms": model, "measured_makespan_ms": meas,
                     "model_over_measured": model / meas, "wall_ms": statistics.median(wall)})
        print(json.dumps(rows[-1]), flush=True)
    out = {"config": args.config, "spec": str(spec), "W_gpu_ms_per_cell_mean": float(cm.W[:, 0].mean()),
           "W_gpu_ms_per_cell_min_max": [float(cm.W[:, 0].min()), float(cm.W[:, 0].max())],
           "W_host_ms_per_cell_1core": float(cm.W[:, 1].mean()), "b_MB_per_ms": cm.b, "rows": rows}
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
