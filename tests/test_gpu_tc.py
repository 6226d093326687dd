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


EDGE = [
    RNNSpec("lstm", 1, 256, 1, 1, algo="tc"),                    # T = 1, B = 1
    RNNSpec("lstm", 2, 64, 5, 1, input=128, dirs=2, algo="tc"),  # smallest TC hidden, bidirectional
    RNNSpec("lstm", 3, 192, 4, 17, input=64, algo="tc"),         # ragged batch (Npad 32), odd depth
    RNNSpec("gru", 1, 256, 6, 128, dtype="bf16"),                # bf16 GRU, full M=128 batch
]


@pytest.mark.parametrize("spec", EDGE, ids=lambda s: f"{s.cell}{s.layers}x{s.hidden}T{s.seq}B{s.batch}d{s.dirs}{s.dtype}")
def test_tc_edge_shapes(spec):
    err = run(spec)
    print(f"edge max-abs {err:.3e}")
    assert err <= (1e-2 if spec.dtype == "bf16" else 1e-4)


def test_tc_initial_states_bidirectional():
    """h0/c0 on the tensor-core path, both directions (state indexing l*D + d)."""
    spec = RNNSpec("lstm", 2, 128, 7, 12, dirs=2, algo="tc")
    w = init_weights(spec, 7)
    x = make_input(spec, 8)
    gen = torch.Generator().manual_seed(11)
    h0 = (torch.rand((4, 12, 128), generator=gen) - 0.5)
    c0 = (torch.rand((4, 12, 128), generator=gen) - 0.5)
    ex = RNNExecutor(spec, w)
    y, hn, cn = ex.forward(x.to(ex.device), h0.to(ex.device), c0.to(ex.device))
    ref = rnn_forward_ref("lstm", x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w],
                          h0.double().numpy(), c0.double().numpy(), dirs=2)
    for g, r in zip((y, hn, cn), ref):
        assert float(np.abs(g.cpu().double().numpy() - r).max()) <= 1e-4


XS_SHAPES = [
    RNNSpec("lstm", 2, 512, 12, 64, input=512, algo="tc"),           # two-group recurrence, layer 0 streamed too
    RNNSpec("lstm", 3, 256, 10, 48, input=512, dirs=2, algo="tc"),   # single-group, bidirectional (D*H = I)
    RNNSpec("gru", 2, 256, 9, 20, input=64, algo="tc"),              # layer 0 not streamed (I != D*H), layer 1 is
    CONFIGS["c2"].with_(seq=40),
]


def test_xp_streaming_forced_matches(tmp_path):
    """XP streaming (the recurrence polls per-M-tile readiness while the rest of
    its K1 runs beside it) forced on with HS_XP_STREAM=1 in a subprocess: outputs
    bit-identical to the default schedule and within 1e-4 of the oracle."""
    import os
    import subprocess
    import sys

    out = tmp_path / "xs.pt"
    code = (
        "import torch, sys; sys.path.insert(0, '.');"
        "from paper_2307_11339_b200 import RNNExecutor, RNNSpec, init_weights, make_input;"
        f"XS_SHAPES = [{', '.join(repr(s) for s in XS_SHAPES)}];"
        "res = [];"
        "[res.append([t.cpu() if t is not None else None for t in RNNExecutor(s, init_weights(s, 0)).forward(make_input(s, 1).cuda())]) for s in XS_SHAPES for _ in range(2)];"
        f"torch.save(res, {str(out)!r})"
    )
    env = dict(os.environ, HS_XP_STREAM="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], env=env, cwd=root, check=True, timeout=600)
    got = torch.load(out)
    for i, spec in enumerate(XS_SHAPES):
        w = init_weights(spec, 0)
        ref = [t.cpu() if t is not None else None for t in RNNExecutor(spec, w).forward(make_input(spec, 1).cuda())]
        for rep in range(2):
            for g, r in zip(got[2 * i + rep], ref):
                assert (g is None and r is None) or torch.equal(g, r), spec
        assert run(spec) <= 1e-4
