"""Tensor-core (tcgen05) path parity against the float64 oracle."""
import numpy as np
import pytest
import torch

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import CONFIGS, RNNExecutor, RNNSpec, init_weights, make_input

pytestmark = pytest.mark.gpu

TC_SHAPES = [
    RNNSpec("lstm", 1, 64, 3, 16, input=64, algo="tc"),
    RNNSpec("lstm", 2, 256, 5, 20, algo="tc"),
    RNNSpec("gru", 2, 128, 6, 8, input=64, dirs=2, algo="tc"),
    RNNSpec("lstm", 2, 512, 9, 64, input=192, dirs=2, algo="tc"),
    RNNSpec("gru", 3, 256, 7, 48, algo="tc"),
    RNNSpec("lstm", 1, 128, 4, 128, algo="tc"),
]


def run(spec, seed=0):
    w = init_weights(spec, seed)
    x = make_input(spec, seed + 1)
    ex = RNNExecutor(spec, w)
    assert ex.algo == "tc"
    y, hn, cn = ex.forward(x.to(ex.device))
    torch.cuda.synchronize()
    ref = rnn_forward_ref(spec.cell, x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w], dirs=spec.dirs)
    got = (y.cpu().double().numpy(), hn.cpu().double().numpy(), None if cn is None else cn.cpu().double().numpy())
    return max(float(np.abs(g - r).max()) for g, r in zip(got, ref) if r is not None)


@pytest.mark.parametrize("spec", TC_SHAPES, ids=lambda s: f"{s.cell}{s.layers}x{s.hidden}T{s.seq}B{s.batch}d{s.dirs}")
def test_tc_shapes(spec):
    err = run(spec)
    print(f"max-abs {err:.3e}")
    assert err <= 1e-4


def test_tc_c2():
    err = run(CONFIGS["c2"].with_(algo="tc"))
    print(f"c2 tc max-abs {err:.3e}")
    assert err <= 1e-4


def test_tc_c3():
    err = run(CONFIGS["c3"].with_(algo="tc"))
    print(f"c3 tc max-abs {err:.3e}")
    assert err <= 1e-4


def test_tc_bf16_mode():
    spec = RNNSpec("lstm", 2, 256, 16, 32, dtype="bf16")
    err = run(spec)
    print(f"bf16 max-abs {err:.3e}")
    assert err <= 1e-2


def test_tc_batch_sliced_bf16():
    """A batch too large for one co-resident recurrence (c5 width, B=200, bf16)
    runs as equal batch slices and still matches the oracle (bf16 budget)."""
    spec = RNNSpec("lstm", 2, 1024, 6, 200, dirs=2, dtype="bf16")
    err = run(spec)
    print(f"sliced bf16 max-abs {err:.3e}")
    assert err <= 1e-2


def test_tc_c5_width_sharded_batch():
    """c5 as one rank of the 8-way request shard sees it: B=32, bf16."""
    err = run(CONFIGS["c5"].with_(seq=12, batch=32))
    print(f"c5 shard bf16 max-abs {err:.3e}")
    assert err <= 1e-2
