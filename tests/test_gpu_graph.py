"""CUDA-graph capture of the device forward (RNNExecutor.graph).

The captured forward runs its layers back to back on one stream; replays on
fresh inputs must equal the eager forward bit for bit (same kernels, tiles
and accumulation order) and the float64 oracle within the north_star
tolerance (max-abs <= 1e-4 fp32, <= 1e-2 bf16)."""
import numpy as np
import pytest
import torch

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import CONFIGS, RNNExecutor, RNNSpec, init_weights, make_input

pytestmark = pytest.mark.gpu

CASES = [
    CONFIGS["c1"],                                           # small-shape cluster kernel
    RNNSpec("lstm", 2, 256, 8, 16, algo="tc"),               # K1 + cluster recurrence, two layers
    RNNSpec("gru", 2, 128, 6, 8, dirs=2, algo="tc"),         # bidirectional
    CONFIGS["c2"].with_(seq=16),                             # two-group recurrence, W_hh in TMEM
    CONFIGS["c3"].with_(seq=24),                             # single-GPU layer wave
    CONFIGS["c4"].with_(layers=2, seq=12),                   # W-streaming ring
    RNNSpec("lstm", 2, 1024, 6, 130, algo="tc"),             # batch slices
    RNNSpec("lstm", 2, 512, 8, 32, dtype="bf16", algo="tc"),
    RNNSpec("lstm", 2, 64, 8, 4),                            # SIMT path
]


@pytest.mark.parametrize("spec", CASES, ids=lambda s: str(s))
def test_graph_replay_matches_eager_and_oracle(spec):
    w = init_weights(spec, 3)
    ex = RNNExecutor(spec, w)
    gf = ex.graph()
    tol = 1e-2 if spec.dtype == "bf16" else 1e-4
    for seed in (11, 12):
        x = make_input(spec, seed)
        y, hn, cn = gf.replay(x.to(ex.device))
        torch.cuda.synchronize()
        ye, hne, cne = ex.forward(x.to(ex.device))
        torch.cuda.synchronize()
        assert torch.equal(y, ye) and torch.equal(hn, hne)
        if cn is not None:
            assert torch.equal(cn, cne)
    ry, rhn, _ = rnn_forward_ref(spec.cell, x.double().numpy(),
                                 [{k: v.double().numpy() for k, v in d.items()} for d in w], dirs=spec.dirs)
    assert float(np.abs(y.cpu().double().numpy() - ry).max()) <= tol
    assert float(np.abs(hn.cpu().double().numpy() - rhn).max()) <= tol
