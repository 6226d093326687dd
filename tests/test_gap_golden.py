"""Replay the reference's archived golden vectors acceptance_out/gap.csv.

The reference regenerates these 200 rows bit-identically.  Here
the corpus is rebuilt with this package's generators, the greedy column with
this package's planner (topo_sort_hybrid + select_devices + evaluate) and the
optimum with the exhaustive oracle (oracle/plan_oracle.py); every float must
match the archived repr exactly.
"""
import csv

import pytest

from oracle.plan_oracle import exhaustive_best, study_corpus
from paper_2307_11339_b200 import costmodel, engine, graph, planner


@pytest.fixture(scope="module")
def rows(golden_dir):
    with open(golden_dir / "reference_gap.csv") as f:
        return list(csv.DictReader(f))


@pytest.fixture(scope="module")
def corpus():
    return study_corpus(200, 42, graph.gen_random_dag, costmodel.SynthParams, costmodel.synth_profile)


def test_corpus_shape_matches(rows, corpus):
    assert len(rows) == len(corpus) == 200
    for r, (g, cm, alpha) in zip(rows, corpus):
        assert int(r["n"]) == g.n and int(r["k"]) == cm.k and float(r["alpha"]) == alpha


def test_greedy_column_bit_exact(rows, corpus):
    for r, (g, cm, alpha) in zip(rows, corpus):
        order = planner.topo_sort_hybrid(g, cm)
        plan = planner.select_devices(g, cm, order, alpha)
        got = engine.evaluate(g, cm, plan).objective
        assert repr(got) == r["greedy_objective"], r["instance"]


def test_oracle_column_bit_exact(rows, corpus):
    for r, (g, cm, alpha) in list(zip(rows, corpus))[::4]:
        best, plan, _ = exhaustive_best(g, cm, alpha, engine, planner.Plan, planner.Order)
        assert repr(best) == r["oracle_objective"], r["instance"]
        greedy = float(r["greedy_objective"])
        assert best <= greedy
        ratio = greedy / best if best > 0 else 1.0
        assert repr(ratio) == r["ratio"]


def test_bruteforce_explored_count_demo7():
    # reference test_oracle.py:69-73: explored = 80 * (1 + k * 2**7) for demo7
    g = graph.gen_demo7()
    cm = costmodel.synth_profile(g, costmodel.SynthParams(k=2), 3)
    _obj, _plan, explored = exhaustive_best(g, cm, 0.0, engine, planner.Plan, planner.Order)
    assert explored == 80 * (1 + 2 * 2**7)
