"""Single-GPU layer wavefront (tc_wave.cuh): every layer's recurrence and
input projection in one cooperative launch, layer l step t beside layer l+1
step t-1 (north_star (b); reference DAG edges graph.py:207-228, dataflow start
rule engine.py:359-372).  Parity against the float64 oracle (fp32 1e-4, bf16
1e-2) on the shapes the wave takes, including ragged batches, initial states,
the maximum layer count, and the host-buffer request path."""
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import CONFIGS, RNNExecutor, RNNSpec, init_weights, make_input

pytestmark = pytest.mark.gpu

WAVE_SHAPES = [
    RNNSpec("gru", 4, 512, 24, 32, algo="tc"),            # c3 width
    RNNSpec("lstm", 2, 256, 9, 20, algo="tc"),             # ragged batch (Npad 32)
    RNNSpec("lstm", 3, 128, 7, 1, input=64, algo="tc"),    # B = 1, I != H (layer-0 K1 with its own K)
    RNNSpec("lstm", 8, 128, 6, 16, algo="tc"),             # the maximum layer count
    RNNSpec("lstm", 4, 256, 17, 48, algo="tc"),            # 3 owner cells per thread, T not a tile multiple
    RNNSpec("gru", 2, 256, 11, 5, input=128, algo="tc"),   # GRU, ragged batch, I != H
]


def oracle(spec, w, x, h0=None, c0=None):
    return rnn_forward_ref(spec.cell, x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w],
                           dirs=spec.dirs,
                           h0=None if h0 is None else h0.double().numpy(),
                           c0=None if c0 is None else c0.double().numpy())


def max_err(got, ref):
    return max(float(np.abs(g.cpu().double().numpy() - r).max()) for g, r in zip(got, ref) if r is not None)


@pytest.mark.parametrize("spec", WAVE_SHAPES, ids=lambda s: f"{s.cell}{s.layers}x{s.hidden}T{s.seq}B{s.batch}")
def test_wave_matches_oracle(spec):
    w = init_weights(spec, 0)
    ex = RNNExecutor(spec, w)
    plan = ex.plan()
    assert plan["layer_wave"], plan
    x = make_input(spec, 1)
    gen = torch.Generator().manual_seed(5)
    shp = (spec.layers, spec.batch, spec.hidden)
    h0 = torch.rand(shp, generator=gen) - 0.5
    c0 = torch.rand(shp, generator=gen) - 0.5 if spec.cell == "lstm" else None
    for states in ((None, None), (h0, c0)):
        dev = ex.device
        got = ex.forward(x.to(dev), *(None if t is None else t.to(dev) for t in states))
        torch.cuda.synchronize()
        err = max_err(got, oracle(spec, w, x, *states))
        print(f"{spec} states={states[0] is not None} plan {plan}: max-abs {err:.3e}")
        assert err <= 1e-4


def test_wave_bf16():
    spec = RNNSpec("lstm", 3, 512, 20, 32, dtype="bf16", algo="tc")
    w = init_weights(spec, 0)
    ex = RNNExecutor(spec, w)
    assert ex.plan()["layer_wave"]
    x = make_input(spec, 1)
    got = ex.forward(x.to(ex.device))
    torch.cuda.synchronize()
    err = max_err(got, oracle(spec, w, x))
    print(f"bf16 wave max-abs {err:.3e}")
    assert err <= 1e-2


def test_wave_repeated_forwards_are_deterministic():
    """Counters and exchange planes are re-zeroed per forward; the K1 claim
    order varies run to run but every tile's sum is fixed, so outputs are
    bit-identical across calls."""
    spec = CONFIGS["c3"].with_(seq=64)
    w = init_weights(spec, 0)
    ex = RNNExecutor(spec, w)
    x = make_input(spec, 1).to(ex.device)
    first = [t.clone() for t in ex.forward(x) if t is not None]
    for _ in range(4):
        again = [t for t in ex.forward(x) if t is not None]
        for a, b in zip(first, again):
            assert torch.equal(a, b)


def test_plan_reports_wave_only_where_it_fits():
    plans = {k: RNNExecutor(CONFIGS[k], init_weights(CONFIGS[k].with_(seq=2), 0)).plan() for k in ("c2", "c3")}
    assert plans["c3"]["layer_wave"] and plans["c3"]["cluster"] == 2
    assert not plans["c2"]["layer_wave"]  # fp32 c2: 2 x 16 MiB of W_hh planes exceed the chip's shared memory


_SUB = r"""
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2307_11339_b200 import CONFIGS, RNNExecutor, init_weights, make_input
spec = CONFIGS["c3"].with_(seq=48)
w = init_weights(spec, 0)
ex = RNNExecutor(spec, w)
y, hn, _ = ex.forward(make_input(spec, 1).to(ex.device))
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([y.cpu().numpy().ravel(), hn.cpu().numpy().ravel()]))
print(ex.plan()["layer_wave"])
"""


def test_wave_agrees_with_layer_by_layer(tmp_path):
    """HS_WAVE=0 (one launch per layer, cluster S=4) vs the wave (S=2): same
    numerics up to the K-split's summation order."""
    outs = {}
    for flag in ("0", "1"):
        f = tmp_path / f"o{flag}.npy"
        env = dict(__import__("os").environ, HS_WAVE=flag)
        r = subprocess.run([sys.executable, "-c", _SUB, str(f)], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        assert r.stdout.strip() == ("True" if flag == "1" else "False")
        outs[flag] = np.load(f)
    d = float(np.abs(outs["0"] - outs["1"]).max())
    print(f"wave vs layer-by-layer max-abs {d:.3e}")
    assert d <= 5e-5
