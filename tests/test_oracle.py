"""The float64 tensor oracle against torch.nn.LSTM / nn.GRU (CPU).

Tensor-side parity is unpinned against the reference (it has no numerics);
the oracle is pinned to PyTorch's documented equations instead, here.
"""
import numpy as np
import pytest
import torch

from oracle.rnn_ref import default_order, grid_node, rnn_forward_ref
from paper_2307_11339_b200 import CONFIGS, RNNSpec, graph, init_weights, make_input, planner, costmodel


def torch_ref(spec, weights, x, h0=None, c0=None):
    mod_cls = torch.nn.LSTM if spec.cell == "lstm" else torch.nn.GRU
    m = mod_cls(spec.I, spec.hidden, spec.layers, bidirectional=spec.dirs == 2).double()
    with torch.no_grad():
        for l in range(spec.layers):
            for d in range(spec.dirs):
                sfx = f"_l{l}" + ("_reverse" if d else "")
                w = weights[l * spec.dirs + d]
                getattr(m, "weight_ih" + sfx).copy_(w["w_ih"].double())
                getattr(m, "weight_hh" + sfx).copy_(w["w_hh"].double())
                getattr(m, "bias_ih" + sfx).copy_(w["b_ih"].double())
                getattr(m, "bias_hh" + sfx).copy_(w["b_hh"].double())
        if spec.cell == "lstm":
            hc = None if h0 is None else (h0.double(), c0.double())
            y, (hn, cn) = m(x.double(), hc)
            return y.numpy(), hn.numpy(), cn.numpy()
        y, hn = m(x.double(), None if h0 is None else h0.double())
        return y.numpy(), hn.numpy(), None


def np_w(weights):
    return [{k: v.numpy() for k, v in w.items()} for w in weights]


@pytest.mark.parametrize(
    "spec",
    [
        CONFIGS["c1"],
        RNNSpec("lstm", 2, 32, 9, 3, input=20),
        RNNSpec("gru", 3, 24, 7, 2, input=16),
        RNNSpec("lstm", 2, 16, 6, 2, dirs=2),
        RNNSpec("gru", 2, 12, 5, 3, input=8, dirs=2),
    ],
)
def test_oracle_matches_torch(spec):
    w = init_weights(spec, seed=3)
    x = make_input(spec, seed=4)
    y, hn, cn = rnn_forward_ref(spec.cell, x.numpy(), np_w(w), dirs=spec.dirs)
    ty, thn, tcn = torch_ref(spec, w, x)
    assert np.abs(y - ty).max() < 1e-12
    assert np.abs(hn - thn).max() < 1e-12
    if cn is not None:
        assert np.abs(cn - tcn).max() < 1e-12


def test_oracle_initial_state():
    spec = RNNSpec("lstm", 2, 16, 5, 3)
    w = init_weights(spec, 1)
    x = make_input(spec, 2)
    g = torch.Generator().manual_seed(9)
    h0 = torch.rand((2, 3, 16), generator=g) - 0.5
    c0 = torch.rand((2, 3, 16), generator=g) - 0.5
    y, hn, cn = rnn_forward_ref("lstm", x.numpy(), np_w(w), h0.numpy(), c0.numpy())
    ty, thn, tcn = torch_ref(spec, w, x, h0, c0)
    assert np.abs(y - ty).max() < 1e-12 and np.abs(cn - tcn).max() < 1e-12


def test_oracle_plan_order_invariant():
    """Evaluating the cells in the planner's hybrid order (Plan.order.seq)
    gives bit-identical tensors to the layer-major order."""
    spec = RNNSpec("lstm", 3, 8, 6, 2)
    g = graph.gen_lstm_grid(spec.layers, spec.seq)
    cm = costmodel.synth_profile(g, costmodel.PRESETS["comm-heavy"], 0)
    order = planner.topo_sort_hybrid(g, cm).seq
    assert list(order) != default_order(3, 6, 1)
    w = np_w(init_weights(spec, 0))
    x = make_input(spec).numpy()
    a = rnn_forward_ref("lstm", x, w)
    b = rnn_forward_ref("lstm", x, w, order=order)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_oracle_rejects_non_topological_order():
    spec = RNNSpec("gru", 2, 8, 3, 1)
    w = np_w(init_weights(spec, 0))
    x = make_input(spec).numpy()
    bad = [grid_node(1, 0, 0, 3, 1)] + [v for v in default_order(2, 3, 1) if v != 3]
    with pytest.raises(ValueError):
        rnn_forward_ref("gru", x, w, order=bad)


def test_bidirectional_grid_orders_are_valid_for_oracle():
    spec = RNNSpec("lstm", 2, 8, 4, 2, dirs=2)
    g = graph.gen_bilstm_grid(2, 4)
    assert graph.validate(g).ok
    order = planner.topo_sort_bfs(g).seq
    w = np_w(init_weights(spec, 0))
    x = make_input(spec).numpy()
    a = rnn_forward_ref("lstm", x, w, dirs=2)
    b = rnn_forward_ref("lstm", x, w, dirs=2, order=order)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
