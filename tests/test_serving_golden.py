"""Serving accounting parity with the reference (servingsim.py:143-288).

`serving_golden.json` holds the metrics.json and events CSVs the reference's
own `hetsched serve` command wrote for each scenario
(tests/golden/make_serving_golden.py).  This package must reproduce them byte
for byte.  The behavioural cases below restate the reference's test intent
(pkg/tests/test_servingsim.py) against this package's API.
"""
import json
from pathlib import Path

import pytest

from paper_2307_11339_b200.serving import (
    ModelEntry,
    Scenario,
    ScenarioError,
    Workload,
    compare_patterns,
    events_to_csv,
    load_scenario,
    run_serving,
    save_scenario,
    slo_from_latency,
)

GOLDEN = json.loads((Path(__file__).parent / "golden" / "serving_golden.json").read_text())


def _metrics_doc(res):
    m = res.metrics
    return {"invocations": m.invocations, "violations": m.violations, "swaps": m.swaps,
            "slo_violation": m.slo_violation, "swapping_rate": m.swapping_rate}


@pytest.mark.parametrize("case", range(len(GOLDEN["cases"])))
def test_serving_matches_reference_cli(case, tmp_path):
    c = GOLDEN["cases"][case]
    f = tmp_path / "scenario.json"
    f.write_text(json.dumps(c["scenario"]))
    sc = load_scenario(f)
    files = {}
    if sc.models is not None:
        res = run_serving(sc.models, sc.capacity_mb, sc.workload, sc.bandwidth_mb_per_ms)
        files["metrics.json"] = json.dumps(_metrics_doc(res), indent=2) + "\n"
        files["events.csv"] = events_to_csv(res.events)
    else:
        rep = compare_patterns(sc.patterns["gpu"], sc.patterns["latency-optimal"], sc.patterns["memory-optimal"],
                               sc.capacity_mb, sc.workload, sc.bandwidth_mb_per_ms)
        files["metrics.json"] = json.dumps(rep.metrics(), indent=2) + "\n"
        for name, res in rep.rows:
            files[f"events-{name}.csv"] = events_to_csv(res.events)
    assert set(files) == set(c["files"])
    for k, v in files.items():
        assert v == c["files"][k], k


def mk(mid, footprint=100.0, exec_ms=10.0, weights=60.0, slo=None):
    return ModelEntry(mid, footprint, exec_ms, weights, slo if slo is not None else slo_from_latency(exec_ms))


def _lat(res):
    return [float(e.detail.split(",")[0].split("=")[1]) for e in res.events if e.event == "complete"]


def test_resident_set_never_swaps():
    res = run_serving([mk(m) for m in "abc"], 1000.0, Workload(9))
    assert res.metrics.swaps == 0
    assert [e.detail for e in res.events if e.event == "load"] == ["cold"] * 3


def test_thrashing_pair_swaps_every_request_after_the_first_two():
    res = run_serving([mk("a", 600.0), mk("b", 600.0)], 1000.0, Workload(20))
    assert res.metrics.swaps == 18 and res.metrics.swapping_rate == 18 / 20
    assert sum(e.event == "evict" for e in res.events) == 19


def test_cold_load_is_the_only_violation():
    m = mk("a", exec_ms=10.0, weights=60.0)  # 5 ms stall at 12 MB/ms against a 12.5 ms SLO
    res = run_serving([m], 1000.0, Workload(8))
    assert res.metrics.violations == 1
    assert _lat(res)[:2] == [15.0, 10.0]


def test_lru_and_fifo_diverge():
    models = [mk(m, 400.0) for m in "abc"]
    w = Workload(6, "random", 31)
    lru, fifo = run_serving(models, 800.0, w), run_serving(models, 800.0, w, policy="fifo")
    assert [e.model for e in lru.events if e.event == "evict"] == ["c", "a"]
    assert [e.model for e in fifo.events if e.event == "evict"] == ["b", "c", "a"]


def test_open_loop_backlog_grows():
    res = run_serving([mk("a", weights=0.0)], 1000.0, Workload(4, interarrival_ms=5.0))
    assert _lat(res) == [10.0, 15.0, 20.0, 25.0]


def test_metrics_recount_and_capacity_invariant():
    models = [mk(m, 350.0) for m in "abcd"]
    res = run_serving(models, 1000.0, Workload(80, "random", 9))
    used, by = 0.0, {m.id: m for m in models}
    for e in res.events:
        used += by[e.model].gpu_footprint_mb if e.event == "load" else -by[e.model].gpu_footprint_mb if e.event == "evict" else 0
        assert used <= 1000.0
    assert res.metrics.swaps == sum(e.event == "load" and e.detail == "swap" for e in res.events)
    assert res.metrics.violations == sum(e.event == "complete" and e.detail.endswith("violation=1") for e in res.events)


@pytest.mark.parametrize("bad", [
    dict(models=[mk("a"), mk("a")]),
    dict(capacity=0.0),
    dict(bandwidth=0.0),
    dict(workload=Workload(0)),
    dict(workload=Workload(3, interarrival_ms=-1.0)),
    dict(models=[mk("a", 2000.0)]),
    dict(models=[mk("a", slo=0.0)]),
    dict(policy="mru"),
    dict(workload=Workload(3, pattern="zipf")),
])
def test_invalid_scenarios_raise(bad):
    kw = dict(models=[mk("a")], capacity=1000.0, workload=Workload(3), bandwidth=12.0, policy="lru")
    kw.update(bad)
    with pytest.raises(ScenarioError):
        run_serving(kw["models"], kw["capacity"], kw["workload"], kw["bandwidth"], kw["policy"])


def test_scenario_round_trip(tmp_path):
    sc = Scenario(1000.0, 12.0, Workload(5, "random", 2, 1.5), models=(mk("a"), mk("b", 300.0)))
    save_scenario(sc, tmp_path / "s.json")
    assert load_scenario(tmp_path / "s.json") == sc
    sp = Scenario(1000.0, 12.0, Workload(5), patterns={"gpu": (mk("a"),), "latency-optimal": (mk("a"),),
                                                       "memory-optimal": (mk("a"),)})
    save_scenario(sp, tmp_path / "p.json")
    assert load_scenario(tmp_path / "p.json") == sp
    (tmp_path / "bad.json").write_text('{"capacity_mb": 1, "bandwidth_mb_per_ms": 1, "workload": {"total_requests": 1}}')
    with pytest.raises(ScenarioError):
        load_scenario(tmp_path / "bad.json")
    with pytest.raises(ScenarioError):
        Scenario(1.0, 1.0, Workload(1))
