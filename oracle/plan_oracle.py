"""Exhaustive plan search for tiny DAGs — TEST INFRASTRUCTURE ONLY.

A restatement of the reference's brute-force optimum
(/root/reference/pkg/src/hetsched/oracle.py:46-189) and its seeded study
corpus (oracle.py:273-300), used by tests/test_gap_golden.py to replay the
reference's archived golden vectors ``acceptance_out/gap.csv`` (copied to
tests/golden/reference_gap.csv): 200 (greedy, optimal) objective pairs.

Search space, as in the reference: every topological order (lexicographic),
every host budget k' in 0..k, every class assignment; a host node takes the
core where it finishes earliest (lowest id on ties).  The first strictly
better candidate wins; the reported objective is the re-evaluated one.
Only the ``engine`` evaluation helpers of the package under test are used for
the per-node recurrence, so the search shares its float arithmetic.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["topological_orders", "exhaustive_best", "study_corpus"]


def topological_orders(graph):
    """All topological orders in lexicographic order."""
    n = graph.n
    indeg = [len(p) for p in graph.pred]
    prefix: list[int] = []

    def rec(ready):
        if len(prefix) == n:
            yield tuple(prefix)
            return
        for u in sorted(ready):
            nxt = set(ready)
            nxt.discard(u)
            prefix.append(u)
            for v in graph.succ[u]:
                indeg[v] -= 1
                if indeg[v] == 0:
                    nxt.add(v)
            yield from rec(nxt)
            for v in graph.succ[u]:
                indeg[v] += 1
            prefix.pop()

    yield from rec({v for v in range(n) if indeg[v] == 0})


def exhaustive_best(graph, cm, alpha, engine, Plan, Order, io_transfers=False, max_nodes=8):
    """(best objective re-evaluated, best plan, candidates explored)."""
    if graph.n > max_nodes:
        raise ValueError(f"instance has {graph.n} nodes, above the enumeration cap {max_nodes}")
    W = cm.W.tolist()
    mem = cm.Mem.tolist()
    inc = cm.incoming
    b = float(cm.b)
    n = graph.n
    pred = graph.pred
    entries = set(graph.entries)
    base = [mem[v][1] + mem[v][2] + mem[v][3] for v in range(n)]
    best = {"obj": math.inf, "cand": None, "count": 0}

    for seq in topological_orders(graph):
        for kp in range(cm.k + 1):
            free = [0.0] * (kp + 1)
            aft = [0.0] * n
            cls = [0] * n
            cores = [0] * n

            def place(pos, macc):
                if pos == n:
                    best["count"] += 1
                    lat = 0.0
                    for v in graph.exits:
                        t = engine._exit_latency(aft[v], mem[v], b, cls[v], io_transfers)
                        if t > lat:
                            lat = t
                    obj = lat + alpha * macc
                    if obj < best["obj"]:
                        best["obj"] = obj
                        best["cand"] = (seq, kp, tuple(cls), tuple(cores))
                    return
                v = seq[pos]
                for c in (0, 1):
                    if c == 1 and kp == 0:
                        continue
                    if c == 0:
                        procs, w = (0,), W[v][0]
                        dm = base[v]
                        for m in pred[v]:
                            if cls[m] != 0:
                                dm += mem[m][1]
                    else:
                        procs, w, dm = range(1, kp + 1), W[v][kp], 0.0
                    rdy = engine._input_ready(mem[v], b, c, v in entries, io_transfers)
                    pj, pf = -1, 0.0
                    for j in procs:
                        _s, f = engine.step_times(pred[v], aft, cls, c, inc[v], b, free[j], w, rdy)
                        if pj < 0 or f < pf:
                            pj, pf = j, f
                    keep = free[pj]
                    cls[v], cores[v], aft[v] = c, pj, pf
                    free[pj] = pf
                    place(pos + 1, macc + dm)
                    free[pj] = keep
                cls[v], cores[v], aft[v] = 0, 0, 0.0

            place(0, 0.0)
    seq, kp, c, cores = best["cand"]
    plan = Plan(order=Order(seq=seq), selection=c, cores=cores, k_star=kp, alpha=alpha)
    return engine.evaluate(graph, cm, plan, io_transfers).objective, plan, best["count"]


def study_corpus(count, seed, gen_random_dag, SynthParams, synth_profile, max_nodes=7, max_k=4,
                 alphas=(0.0, 0.25, 1.0)):
    """The reference's seeded gap-study corpus (oracle.py:273-300): same draw
    sequence, so ``study_corpus(200, 42)`` rebuilds the archived instances."""
    rng = np.random.default_rng(seed)
    out = []
    for idx in range(count):
        n = int(rng.integers(4, max_nodes + 1))
        p = 0.4 + 0.3 * float(rng.random())
        k = int(rng.integers(1, max_k + 1))
        g = gen_random_dag(n, p, int(rng.integers(0, 2**31)))
        params = SynthParams(
            gpu_mean=4.0 + 8.0 * float(rng.random()),
            cpu_base_mean=4.0 + 8.0 * float(rng.random()),
            contention_slope=0.05 + 0.15 * float(rng.random()),
            comm_mean=1.0 + 6.0 * float(rng.random()),
            b=4.0,
            k=k,
        )
        cm = synth_profile(g, params, int(rng.integers(0, 2**31)))
        out.append((g, cm, alphas[idx % len(alphas)]))
    return out
