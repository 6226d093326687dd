"""Plan execution (drop-in for engine.simulate) and the measured profiler
(drop-in for synth_profile): host-side logic on CPU, hybrid/fused parity on GPU.

Tolerance: max-abs <= 1e-4 against the float64 oracle (BASELINE north_star).
"""
import numpy as np
import pytest
import torch

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import (
    RNNSpec,
    costmodel,
    engine,
    graph,
    init_weights,
    make_input,
    planner,
)
from paper_2307_11339_b200.executor import HostRNN, build_schedule, check_grid, execute, profile_ops
from paper_2307_11339_b200.planner import Order, Plan

TOL = 1e-4

SPECS = [
    RNNSpec("lstm", 2, 24, 7, 3),
    RNNSpec("gru", 3, 16, 6, 2, input=8),
    RNNSpec("lstm", 2, 12, 5, 2, dirs=2),
    RNNSpec("gru", 2, 8, 4, 3, input=4, dirs=2),
]
IDS = [f"{s.cell}{s.layers}x{s.hidden}T{s.seq}d{s.dirs}" for s in SPECS]


def grid_of(spec):
    return graph.gen_lstm_grid(spec.layers, spec.seq) if spec.dirs == 1 else graph.gen_bilstm_grid(spec.layers, spec.seq)


def random_plan(g, seed, k_star=3, p_gpu=0.5, order=None):
    rng = np.random.default_rng(seed)
    if order is None:
        order = planner.topo_sort_bfs(g) if seed % 2 else planner.topo_sort_dfs(g)
    sel = tuple(int(x) for x in (rng.random(g.n) >= p_gpu))
    cores = tuple(int(rng.integers(1, k_star + 1)) if s else 0 for s in sel)
    return Plan(order=order, selection=sel, cores=cores, k_star=k_star if any(sel) else 0, alpha=0.0)


def oracle(spec, w, x, h0=None, c0=None):
    return rnn_forward_ref(
        spec.cell, x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w],
        None if h0 is None else h0.double().numpy(), None if c0 is None else c0.double().numpy(), dirs=spec.dirs,
    )


def err(res, ref):
    got = (res.y, res.hn, res.cn)
    return max(float(np.abs(g.detach().cpu().double().numpy() - r).max()) for g, r in zip(got, ref) if r is not None)


# --------------------------------------------------------------- CPU tier
@pytest.mark.parametrize("spec", SPECS, ids=IDS)
def test_schedule_covers_plan(spec):
    g = grid_of(spec)
    for seed in range(20):
        plan = random_plan(g, seed)
        sc = build_schedule(g, plan, spec)
        gpu_nodes = [v for seg in sc.gpu for v in seg.nodes]
        assert sorted(gpu_nodes) == [v for v in range(g.n) if plan.selection[v] == 0]
        pos = {v: i for i, v in enumerate(plan.order.seq)}
        for seg in sc.gpu:
            assert seg.s1 - seg.s0 == len(seg.nodes)
            for i, v in enumerate(seg.nodes):
                l, d, t, s = sc.cells[v]
                assert l * spec.dirs + d == seg.ld and s == seg.s0 + i
                if i:  # only the first node of a segment may wait on host cells
                    assert all(plan.selection[m] == 0 for m in g.pred[v])
        # GPU queue keeps plan order
        firsts = [pos[seg.nodes[0]] for seg in sc.gpu]
        assert firsts == sorted(firsts)
        for core, q in sc.host.items():
            assert all(plan.cores[v] == core and plan.selection[v] == 1 for v in q)
            assert [pos[v] for v in q] == sorted(pos[v] for v in q)


def test_schedule_merges_all_gpu_layer():
    spec = RNNSpec("lstm", 2, 8, 6, 1)
    g = grid_of(spec)
    plan = Plan(order=planner.topo_sort_bfs(g), selection=(0,) * g.n, cores=(0,) * g.n, k_star=0, alpha=0.0)
    # BFS interleaves layers, so segments alternate; DFS-by-layer order gives one per layer
    seq = tuple(range(g.n))
    plan2 = Plan(order=Order(seq), selection=(0,) * g.n, cores=(0,) * g.n, k_star=0, alpha=0.0)
    assert len(build_schedule(g, plan2, spec).gpu) == 2
    assert sum(len(s.nodes) for s in build_schedule(g, plan, spec).gpu) == g.n


def test_check_grid_rejects_other_graphs():
    spec = RNNSpec("lstm", 2, 8, 4, 1)
    with pytest.raises(ValueError):
        check_grid(graph.gen_lstm_grid(2, 5), spec)
    with pytest.raises(ValueError):
        check_grid(graph.gen_random_dag(8, 0.3, 0), spec)
    check_grid(graph.gen_lstm_grid(2, 4), spec)


def test_plan_validation():
    spec = RNNSpec("lstm", 1, 8, 4, 1)
    g = grid_of(spec)
    bad_order = Plan(order=Order((1, 0, 2, 3)), selection=(1,) * 4, cores=(1,) * 4, k_star=1, alpha=0.0)
    with pytest.raises(ValueError):
        build_schedule(g, bad_order, spec)
    bad_core = Plan(order=Order((0, 1, 2, 3)), selection=(1,) * 4, cores=(2,) * 4, k_star=1, alpha=0.0)
    with pytest.raises(ValueError):
        build_schedule(g, bad_core, spec)


@pytest.mark.parametrize("spec", SPECS, ids=IDS)
def test_all_host_plan_matches_oracle(spec):
    """The reference's CPU pattern (every cell on host cores, k* workers)."""
    g = grid_of(spec)
    w = init_weights(spec, 3)
    x = make_input(spec, 4)
    host = HostRNN(spec, w)
    ref = oracle(spec, w, x)
    for seed in range(3):
        plan = random_plan(g, seed, k_star=1 + seed, p_gpu=0.0)
        res = execute(g, plan, host, x)
        assert err(res, ref) <= TOL
        assert sorted(s.node for s in res.trace.nodes) == list(range(g.n))
        assert res.trace.transfers == ()
        # the reference's makespan: last node end (engine.py:408-415); wall_ms adds the assembly
        assert res.trace.makespan == max(s.end for s in res.trace.nodes) <= res.wall_ms
        # each core runs its cells one at a time, in plan order
        pos = {v: i for i, v in enumerate(plan.order.seq)}
        for core in set(plan.cores):
            sp = sorted((s for s in res.trace.nodes if s.device == core), key=lambda s: pos[s.node])
            assert all(a.end <= b.start for a, b in zip(sp, sp[1:]))


def test_all_host_plan_initial_states():
    spec = RNNSpec("lstm", 2, 10, 5, 2)
    g = grid_of(spec)
    w = init_weights(spec, 1)
    x = make_input(spec, 2)
    gen = torch.Generator().manual_seed(9)
    h0 = torch.rand((2, 2, 10), generator=gen) - 0.5
    c0 = torch.rand((2, 2, 10), generator=gen) - 0.5
    plan = random_plan(g, 1, k_star=2, p_gpu=0.0)
    res = execute(g, plan, HostRNN(spec, w), x, h0, c0)
    assert err(res, oracle(spec, w, x, h0, c0)) <= TOL


def test_gpu_plan_needs_executor():
    spec = RNNSpec("lstm", 1, 8, 4, 1)
    g = grid_of(spec)
    plan = Plan(order=Order((0, 1, 2, 3)), selection=(0,) * 4, cores=(0,) * 4, k_star=0, alpha=0.0)
    with pytest.raises(ValueError):
        execute(g, plan, HostRNN(spec, init_weights(spec)), make_input(spec))


def test_profile_host_model_tables():
    spec = RNNSpec("lstm", 2, 16, 6, 2, input=8)
    g = grid_of(spec)
    cm = profile_ops(g, HostRNN(spec, init_weights(spec)), k=2, reps=2)
    costmodel.check_compatible(g, cm)
    assert cm.W.shape == (g.n, 3) and cm.k == 2
    assert np.all(cm.W[:, 0] > cm.W[:, 1])  # no GPU: never placed there
    # state edges carry h and c, layer edges carry h
    B, H = spec.batch, spec.hidden
    assert cm.C[0, 1] == 2 * B * H * 4 / 2**20
    assert cm.C[0, spec.seq] == B * H * 4 / 2**20
    assert np.array_equal(cm.Mem, costmodel.snap_mem(cm.Mem))
    plan = planner.latency_optimal_plan(g, cm)
    assert all(s == 1 for s in plan.selection)
    res = execute(g, plan, HostRNN(spec, init_weights(spec)), make_input(spec))
    assert err(res, oracle(spec, init_weights(spec), make_input(spec))) <= TOL


# --------------------------------------------------------------- GPU tier
@pytest.mark.gpu
@pytest.mark.parametrize("spec", SPECS, ids=IDS)
def test_hybrid_plans_match_oracle(spec):
    from paper_2307_11339_b200 import RNNExecutor

    g = grid_of(spec)
    w = init_weights(spec, 5)
    x = make_input(spec, 6)
    ex = RNNExecutor(spec, w)
    ref = oracle(spec, w, x)
    for seed in range(4):
        plan = random_plan(g, seed, k_star=2, p_gpu=0.5)
        res = execute(g, plan, ex, x)
        e = err(res, ref)
        assert e <= TOL, f"seed {seed}: max-abs {e}"
        assert res.y.device.type == "cuda"
        assert sorted(s.node for s in res.trace.nodes) == list(range(g.n))
        crossings = sum((plan.selection[a] == 0) != (plan.selection[b] == 0) for a, b in g.edge_set)
        if crossings:
            assert res.trace.transfers


@pytest.mark.gpu
def test_all_gpu_plan_is_fused_forward():
    from paper_2307_11339_b200 import CONFIGS, RNNExecutor

    spec = CONFIGS["c2"].with_(seq=32)
    g = grid_of(spec)
    w = init_weights(spec)
    x = make_input(spec)
    ex = RNNExecutor(spec, w)
    plan = Plan(order=planner.topo_sort_bfs(g), selection=(0,) * g.n, cores=(0,) * g.n, k_star=0, alpha=0.0)
    res = execute(g, plan, ex, x)
    y, hn, cn = ex.forward(x.to(ex.device))
    assert torch.equal(res.y, y) and torch.equal(res.hn, hn) and torch.equal(res.cn, cn)
    assert len(res.trace.nodes) == g.n and res.trace.makespan > 0
    assert abs(res.trace.makespan - max(sp.end for sp in res.trace.nodes)) < 1e-9  # engine.py:408-415
    assert res.wall_ms >= res.trace.makespan


@pytest.mark.gpu
def test_profile_plan_execute_c1():
    """c1 end to end: measured profile -> latency-optimal plan -> execute."""
    from paper_2307_11339_b200 import CONFIGS, RNNExecutor

    spec = CONFIGS["c1"]
    g = grid_of(spec)
    w = init_weights(spec)
    x = make_input(spec)
    ex = RNNExecutor(spec, w)
    cm = profile_ops(g, ex, k=2, reps=3)
    costmodel.check_compatible(g, cm)
    assert np.all(cm.W > 0) and cm.b > 5  # pinned H2D, MB/ms (= GB/s); PCIe Gen5 x16 measures ~50
    plan = planner.latency_optimal_plan(g, cm)
    res = execute(g, plan, ex, x)
    assert err(res, oracle(spec, w, x)) <= TOL
    gpu_plan, cpu_plan = engine.baseline_plans(g, cm)
    for p in (gpu_plan, cpu_plan):
        assert err(execute(g, p, ex, x), oracle(spec, w, x)) <= TOL
