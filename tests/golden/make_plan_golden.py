"""Generate tests/golden/plan_golden.json from the REFERENCE planner itself.

Run in the build container only (needs /root/reference):
    python tests/golden/make_plan_golden.py

It imports the unmodified reference package (hetsched, from
/root/reference/pkg/src) and records, for a fixed corpus of graphs/profiles,
the reference's orders, plans, evaluations, core-count sweeps, movement
passes, baselines and simulated makespans.  tests/test_plan_parity.py replays
the corpus through paper_2307_11339_b200 and requires bit-exact equality.
The corpus is rebuilt with the same generators on both sides (their draw
sequences are part of what is checked).
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).with_name("plan_golden.json")


def h(obj) -> str:
    return hashlib.sha256(repr(obj).encode()).hexdigest()[:24]


def corpus_specs():
    """(kind, args, preset_or_params, seed) tuples — interpreted identically by
    the replay test."""
    specs = []
    for preset in ("gpu-dominant", "cpu-comparable", "comm-heavy"):
        for seed in (0, 5, 11):
            specs.append(("demo7", [], preset, seed))
    for L, T in ((1, 16), (2, 4), (4, 8), (3, 4), (2, 128), (4, 64), (8, 16)):
        for preset in ("cpu-comparable", "gpu-dominant", "comm-heavy"):
            specs.append(("lstm", [L, T], preset, 0))
    specs.append(("lstm", [4, 256], "cpu-comparable", 0))
    specs.append(("lstm", [8, 512], "cpu-comparable", 0))  # c4 grid (n = 4096)
    rng = np.random.default_rng(2026)
    for _ in range(40):
        n = int(rng.integers(2, 40))
        p = float(0.05 + 0.5 * rng.random())
        gseed = int(rng.integers(0, 2**31))
        params = {
            "gpu_mean": float(2.0 + 10.0 * rng.random()),
            "cpu_base_mean": float(2.0 + 10.0 * rng.random()),
            "contention_slope": float(0.2 * rng.random()),
            "comm_mean": float(0.5 + 5.0 * rng.random()),
            "b": float(1.0 + 7.0 * rng.random()),
            "k": int(rng.integers(1, 6)),
        }
        specs.append(("random", [n, p, gseed], params, int(rng.integers(0, 2**31))))
    return specs


def build(mod_graph, mod_cost, kind, args, prof, seed):
    if kind == "demo7":
        g = mod_graph.gen_demo7()
    elif kind == "lstm":
        g = mod_graph.gen_lstm_grid(*args)
    else:
        g = mod_graph.gen_random_dag(*args)
    params = mod_cost.PRESETS[prof] if isinstance(prof, str) else mod_cost.SynthParams(**prof)
    return g, mod_cost.synth_profile(g, params, seed)


class _Stuck(Exception):
    pass


def _bounded_moves(planner, g, cm, plan, io):
    """The reference's reduce_movements can cycle forever when two flips keep
    an equal objective (e.g. gen_lstm_grid(2, 4), cpu-comparable): give it
    2 s and record None ("does not terminate") in that case."""
    import signal

    def on_alarm(*_):
        raise _Stuck()

    old = signal.signal(signal.SIGALRM, on_alarm)
    signal.setitimer(signal.ITIMER_REAL, 2.0)
    try:
        return planner.reduce_movements(g, cm, plan, None, io)
    except _Stuck:
        return None
    finally:
        signal.setitimer(signal.ITIMER_REAL, 0)
        signal.signal(signal.SIGALRM, old)


def record(hs, g, cm):
    from hetsched import engine, planner

    rec = {"n": g.n, "edges_hash": h(sorted(g.edge_set))}
    rec["bfs"] = list(planner.topo_sort_bfs(g).seq)
    rec["dfs"] = list(planner.topo_sort_dfs(g).seq)
    order = planner.topo_sort_hybrid(g, cm)
    rec["hybrid"] = list(order.seq)
    rec["cases"] = []
    big = g.n > 300
    for alpha in ((0.0, 1.0) if big else (0.0, 0.25, 1.0, 3.0)):
        for io in ((False,) if big else (False, True)):
            pts = planner.sweep_core_counts(g, cm, order, alpha, io)
            plan = planner.select_devices(g, cm, order, alpha, io)
            ev = engine.evaluate(g, cm, plan, io)
            sim = engine.simulate(g, cm, plan, False, io)
            simc = engine.simulate(g, cm, plan, True, io) if not big else sim
            mv = _bounded_moves(planner, g, cm, plan, io) if g.n <= 64 else plan
            rec["cases"].append({
                "alpha": alpha, "io": io,
                "points": [[p.k_prime, p.latency, p.gpu_memory, p.total_cost, list(p.plan.selection), list(p.plan.cores)] for p in pts],
                "selection": list(plan.selection), "cores": list(plan.cores), "k_star": plan.k_star,
                "latency": ev.latency, "gpu_memory": ev.gpu_memory, "objective": ev.objective,
                "est_hash": h(ev.est), "aft_hash": h(ev.aft),
                "sim_makespan": sim.makespan, "sim_csv_hash": h(engine.trace_to_csv(sim)),
                "simc_makespan": simc.makespan, "simc_csv_hash": h(engine.trace_to_csv(simc)),
                "moves_selection": list(mv.selection) if mv else None,
                "moves_cores": list(mv.cores) if mv else None,
                "moves_checked": g.n <= 64,
            })
    gp, cp = engine.baseline_plans(g, cm)
    rec["baseline_cpu"] = [list(cp.cores), cp.k_star]
    rec["baseline_gpu_latency"] = engine.evaluate(g, cm, gp).latency
    return rec


def main():
    sys.path.insert(0, str(REF))
    import hetsched
    from hetsched import costmodel, graph

    out = {"generator": "tests/golden/make_plan_golden.py", "reference": "hetsched " + hetsched.__version__, "instances": []}
    for spec in corpus_specs():
        g, cm = build(graph, costmodel, *spec)
        r = record(hetsched, g, cm)
        r["spec"] = list(spec)
        out["instances"].append(r)
    OUT.write_text(json.dumps(out, separators=(",", ":")) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(out['instances'])} instances)")


if __name__ == "__main__":
    main()
