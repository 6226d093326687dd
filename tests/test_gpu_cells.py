"""Cell-level GPU entry points: hybrid-plan segments on the tensor-core path
(hs_rnn_run_cells) and the per-cell profiler (hs_rnn_profile_cells, the
measured W[:, 0] of costmodel.synth_profile, costmodel.py:176-221).

Tolerance: max-abs <= 1e-4 against the float64 oracle (north_star)."""
import numpy as np
import pytest
import torch

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import RNNExecutor, RNNSpec, graph, init_weights, make_input, planner
from paper_2307_11339_b200.executor import execute, profile_ops
from paper_2307_11339_b200.planner import Plan

pytestmark = pytest.mark.gpu
TOL = 1e-4

TC_SPECS = [
    RNNSpec("lstm", 2, 128, 8, 16, algo="tc"),
    RNNSpec("gru", 2, 256, 6, 8, dirs=2, algo="tc"),
    RNNSpec("lstm", 2, 128, 7, 4, input=64, dirs=2, algo="tc"),
]
IDS = [f"{s.cell}{s.layers}x{s.hidden}T{s.seq}B{s.batch}d{s.dirs}" for s in TC_SPECS]


def oracle(spec, w, x):
    return rnn_forward_ref(spec.cell, x.double().numpy(),
                           [{k: v.double().numpy() for k, v in d.items()} for d in w], dirs=spec.dirs)


def grid_of(spec):
    return graph.gen_lstm_grid(spec.layers, spec.seq) if spec.dirs == 1 else graph.gen_bilstm_grid(spec.layers, spec.seq)


@pytest.mark.parametrize("spec", TC_SPECS, ids=IDS)
def test_segments_on_tensor_cores_compose_to_the_forward(spec):
    """Each layer-direction run as two segments through hs_rnn_run_cells
    (split + K1 + one recurrence launch each, reverse direction included)
    reproduces the fused forward and the oracle."""
    w = init_weights(spec, 2)
    x = make_input(spec, 3).cuda()
    ex = RNNExecutor(spec, w)
    assert ex.algo == "tc"
    y_f, hn_f, cn_f = ex.forward(x)
    T, B, H, D = spec.seq, spec.batch, spec.hidden, spec.dirs
    inp = x
    hn = torch.empty_like(hn_f)
    cn = torch.empty_like(hn_f)
    for l in range(spec.layers):
        out = torch.zeros((T, B, D * H), device="cuda")
        for d in range(D):
            ld = l * D + d
            h = torch.zeros((B, H), device="cuda")
            c = torch.zeros((B, H), device="cuda")
            cut = T // 2 + 1
            for t0, t1 in ((0, cut), (cut, T)):
                h2, c2 = torch.empty_like(h), torch.empty_like(c)
                ex.run_cells(ld, t0, t1, inp, out, h, c if spec.cell == "lstm" else None, h2,
                             c2 if spec.cell == "lstm" else None)
                assert ex.last_launch_count() == 4  # split, K1, zeroing, recurrence: the tensor-core segment
                h, c = h2, c2
            hn[ld], cn[ld] = h, c
        inp = out
    torch.cuda.synchronize()
    assert float((out - y_f).abs().max()) <= 1e-6
    assert float((hn - hn_f).abs().max()) <= 1e-6
    ry, rhn, rcn = oracle(spec, w, x.cpu())
    assert float(np.abs(out.cpu().double().numpy() - ry).max()) <= TOL
    if spec.cell == "lstm":
        assert float((cn - cn_f).abs().max()) <= 1e-6


SMALL_SPECS = [
    RNNSpec("lstm", 1, 128, 16, 1, algo="simt"),  # BASELINE c1 (auto resolves to this path)
    RNNSpec("gru", 2, 64, 9, 4, dirs=2, algo="simt"),
    RNNSpec("lstm", 2, 96, 7, 3, input=40, dirs=2, algo="simt"),
]


@pytest.mark.parametrize("spec", SMALL_SPECS, ids=[f"{s.cell}{s.layers}x{s.hidden}T{s.seq}B{s.batch}d{s.dirs}" for s in SMALL_SPECS])
def test_segments_on_the_small_shape_kernel_compose_to_the_forward(spec):
    """Shapes the fused forward runs on the small-shape cluster kernel run
    their hybrid-plan segments on it too (one launch per segment, steps
    s_base.. of the layer, reverse direction included): what profile_ops
    timed for W[:, 0].  Same per-step arithmetic as the fused launch."""
    w = init_weights(spec, 2)
    x = make_input(spec, 3).cuda()
    ex = RNNExecutor(spec, w)
    assert ex.algo == "simt"
    y_f, hn_f, cn_f = ex.forward(x)
    T, B, H, D = spec.seq, spec.batch, spec.hidden, spec.dirs
    inp = x
    hn = torch.empty_like(hn_f)
    cn = torch.empty_like(hn_f)
    for l in range(spec.layers):
        out = torch.zeros((T, B, D * H), device="cuda")
        for d in range(D):
            ld = l * D + d
            h = torch.zeros((B, H), device="cuda")
            c = torch.zeros((B, H), device="cuda")
            for t0, t1 in ((0, 3), (3, T // 2 + 1), (T // 2 + 1, T)):
                h2, c2 = torch.empty_like(h), torch.empty_like(c)
                ex.run_cells(ld, t0, t1, inp, out, h, c if spec.cell == "lstm" else None, h2,
                             c2 if spec.cell == "lstm" else None)
                assert ex.last_launch_count() == 1  # the small-shape cluster kernel alone
                h, c = h2, c2
            hn[ld], cn[ld] = h, c
        inp = out
    torch.cuda.synchronize()
    assert float((out - y_f).abs().max()) <= 1e-6
    assert float((hn - hn_f).abs().max()) <= 1e-6
    if spec.cell == "lstm":
        assert float((cn - cn_f).abs().max()) <= 1e-6
    ry, _rhn, _rcn = oracle(spec, w, x.cpu())
    assert float(np.abs(out.cpu().double().numpy() - ry).max()) <= TOL


@pytest.mark.parametrize("spec", TC_SPECS, ids=IDS)
def test_hybrid_plans_on_tensor_core_segments(spec):
    g = grid_of(spec)
    w = init_weights(spec, 5)
    x = make_input(spec, 6)
    ex = RNNExecutor(spec, w)
    ref = oracle(spec, w, x)
    rng = np.random.default_rng(0)
    for seed in range(3):
        order = planner.topo_sort_bfs(g) if seed % 2 else planner.topo_sort_dfs(g)
        sel = tuple(int(v) for v in (rng.random(g.n) >= 0.5))
        cores = tuple(int(rng.integers(1, 3)) if s else 0 for s in sel)
        plan = Plan(order=order, selection=sel, cores=cores, k_star=2 if any(sel) else 0, alpha=0.0)
        res = execute(g, plan, ex, x)
        got = (res.y, res.hn, res.cn)
        e = max(float(np.abs(a.detach().cpu().double().numpy() - r).max()) for a, r in zip(got, ref) if r is not None)
        assert e <= TOL, f"seed {seed}: {e}"


@pytest.mark.parametrize("spec", [
    RNNSpec("lstm", 2, 1024, 16, 64, algo="tc"),     # two-group recurrence (c2 width)
    RNNSpec("gru", 4, 512, 24, 32, algo="tc"),       # single-GPU layer wavefront (c3 width)
    RNNSpec("lstm", 1, 256, 12, 16, dirs=2, algo="tc"),
    RNNSpec("lstm", 2, 64, 8, 4),                    # SIMT / small-shape path: no stamps, mean period
], ids=["two-group", "wave", "bidir", "simt"])
def test_profile_cells_sums_to_the_forward(spec):
    ex = RNNExecutor(spec, init_weights(spec, 1))
    x = make_input(spec, 2).cuda()
    ex.forward(x)
    cells, fwd = ex.profile_cells(x)
    assert len(cells) == spec.layers * spec.dirs * spec.seq
    assert fwd > 0 and all(c > 0 for c in cells)
    assert abs(sum(cells) - fwd) <= 1e-3 * fwd
    g = grid_of(spec)
    cm = profile_ops(g, ex, k=1, reps=3)
    assert abs(float(cm.W[:, 0].sum()) - fwd) <= 0.3 * fwd  # medians of fresh runs
