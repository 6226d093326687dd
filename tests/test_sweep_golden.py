"""f2: the latency/memory frontier against the reference's own `sweep`.

tests/golden/sweep_golden.json holds sweep.csv files written by the
unmodified reference CLI (tests/golden/make_sweep_golden.py: `hetsched
gen-graph` / `gen-profile` / `sweep`, cli.py:259-306, alpha grid cli.py:125-140).
The same graph and profile are rebuilt here, round-tripped through this
package's JSON I/O like the CLI does, and planner.sweep_csv must produce the
identical text.  Then the memory-optimal chooser the reference lacks
(memory_optimal_alpha) is checked on the frontier.
"""
import json
from pathlib import Path

import pytest

from paper_2307_11339_b200 import costmodel, engine, graph, planner

CASES = json.loads((Path(__file__).parent / "golden" / "sweep_golden.json").read_text())["cases"]


def rebuild(case, tmp_path):
    a = case["graph_args"]
    fam = a[a.index("--family") + 1]
    opt = lambda k, d: a[a.index(k) + 1] if k in a else d  # noqa: E731
    if fam == "lstm":
        g = graph.gen_lstm_grid(int(opt("--layers", 2)), int(opt("--seq", 8)))
    elif fam == "demo7":
        g = graph.gen_demo7()
    else:
        g = graph.gen_random_dag(int(opt("--nodes", 16)), float(opt("--edge-prob", 0.3)), int(opt("--seed", 0)))
    graph.save_graph(g, tmp_path / "graph.json")
    g = graph.load_graph(tmp_path / "graph.json")
    cm = costmodel.synth_profile(g, costmodel.PRESETS[case["preset"]], case["profile_seed"])
    costmodel.save_profile(cm, tmp_path / "profile.json")
    return g, costmodel.load_profile(tmp_path / "profile.json")


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_sweep_csv_matches_reference(idx, tmp_path):
    case = CASES[idx]
    g, cm = rebuild(case, tmp_path)
    assert planner.sweep_csv(g, cm, case["alphas"], case["io_transfers"]) == case["sweep_csv"]


def _rows(text):
    rows = [r.split(",") for r in text.strip().split("\n")[1:]]
    return [(k, float(a) if a else None, float(lat), float(mem), int(ks)) for k, a, lat, mem, ks in rows]


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_memory_optimal_alpha_on_reference_frontier(idx, tmp_path):
    """Default SLO = the all-GPU pattern's latency: the chosen point meets it
    and no frontier point that meets it uses less GPU memory; ties go to the
    larger alpha."""
    case = CASES[idx]
    g, cm = rebuild(case, tmp_path)
    rows = _rows(case["sweep_csv"])
    plans = [r for r in rows if r[0] == "plan"]
    slo = next(r[2] for r in rows if r[0] == "baseline-gpu")
    best = planner.memory_optimal_alpha(g, cm, None, case["alphas"], case["io_transfers"])
    feasible = [r for r in plans if r[2] <= slo]
    if not feasible:
        assert best.alpha == plans[0][1]
        return
    assert best.latency <= slo
    assert best.gpu_memory == min(r[3] for r in feasible)
    assert best.alpha == max(r[1] for r in feasible if r[3] == best.gpu_memory)


def test_memory_optimal_alpha_slo_edges(tmp_path):
    g, cm = rebuild(CASES[2], tmp_path)  # c2 grid, cpu-comparable
    pts = planner.sweep_alpha(g, cm, "0:1:0.1")
    # an SLO below every point: fall back to the latency-optimal (alpha = 0) point
    low = planner.memory_optimal_alpha(g, cm, min(p.latency for p in pts) * 0.5, "0:1:0.1")
    assert low.alpha == 0.0
    # an SLO above every point: the least GPU memory on the whole frontier
    high = planner.memory_optimal_alpha(g, cm, max(p.latency for p in pts) * 2, "0:1:0.1")
    assert high.gpu_memory == min(p.gpu_memory for p in pts)
    # the SLO exactly at a point's latency admits that point (<=)
    p = pts[3]
    at = planner.memory_optimal_alpha(g, cm, p.latency, "0:1:0.1")
    assert at.latency <= p.latency and at.gpu_memory <= p.gpu_memory
    with pytest.raises(ValueError):
        planner.sweep_alpha(g, cm, "1:0:0.1")


def test_memory_optimal_plan_executes_within_slo_model(tmp_path):
    """The chosen plan re-evaluates to the frontier's numbers (engine.evaluate)."""
    g, cm = rebuild(CASES[0], tmp_path)
    best = planner.memory_optimal_alpha(g, cm)
    ev = engine.evaluate(g, cm, best.plan)
    assert (ev.latency, ev.gpu_memory) == (best.latency, best.gpu_memory)
