"""Full-size parity on the BASELINE configs against committed float64 goldens.

tests/golden/tensor_c{2..5}.npz hold the float64 oracle's outputs (sampled:
final states of every layer-direction and y at three timesteps, for the batch
rows tensor_sample.py lists), made offline by tests/golden/make_tensor_golden.py.
Each test runs the full BASELINE config — full T, all layers, full batch —
through the C ABI and compares every stored entry.

Tolerances (written here, per BASELINE.json north_star):
  fp32 mode  max-abs <= 1e-4  (c2, c3, c4)
  bf16 mode  max-abs <= 1e-2  (c5, opt-in)
"""
import sys

import numpy as np
import pytest
import torch

from paper_2307_11339_b200 import CONFIGS, RNNExecutor, init_weights, make_input

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent / "golden"))
from tensor_sample import sample_index, take  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 1e-2}


def compare(gold, y, hn, cn, T, B, rows=None):
    """max-abs over the stored entries; ``rows`` restricts to the first rows of
    the batch sample (a shard run on a batch prefix)."""
    ys, hs, cs = take(y, hn, cn, T, B)
    gy, gh = gold["y"], gold["hn"]
    gc = gold["cn"] if "cn" in gold.files else None
    if rows is not None:
        gy, gh = gy[:, :rows], gh[:, :rows]
        gc = None if gc is None else gc[:, :rows]
    errs = {"y": float(np.abs(ys.cpu().double().numpy() - gy).max()),
            "hn": float(np.abs(hs.cpu().double().numpy() - gh).max())}
    if gc is not None:
        errs["cn"] = float(np.abs(cs.cpu().double().numpy() - gc).max())
    return errs


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_size_matches_golden(name, golden_dir):
    spec = CONFIGS[name]
    gold = np.load(golden_dir / f"tensor_{name}.npz")
    ts, bs = sample_index(spec.seq, spec.batch)
    assert list(gold["ts"]) == ts and list(gold["bs"]) == bs
    ex = RNNExecutor(spec, init_weights(spec, 0))
    x = make_input(spec, 1).to(ex.device)
    y, hn, cn = ex.forward(x)
    torch.cuda.synchronize()
    errs = compare(gold, y, hn, cn, spec.seq, spec.batch)
    print(f"{name} full size ({spec.layers}x{spec.hidden} T{spec.seq} B{spec.batch} d{spec.dirs} {spec.dtype}, "
          f"plan {ex.plan()}): max-abs {errs}")
    assert max(errs.values()) <= TOL[spec.dtype], errs


def test_c5_request_shard_matches_golden(golden_dir):
    """c5 as one rank of the 8-way request shard runs it: the first 32 sequences
    of the same request (B=32, full T=1024, 3 bidirectional layers, bf16)."""
    spec = CONFIGS["c5"]
    gold = np.load(golden_dir / "tensor_c5.npz")
    shard = spec.with_(batch=32)
    ex = RNNExecutor(shard, init_weights(spec, 0))
    x = make_input(spec, 1)[:, :32].contiguous().to(ex.device)
    y, hn, cn = ex.forward(x)
    torch.cuda.synchronize()
    ts, _ = sample_index(spec.seq, spec.batch)
    ys, hs, cs = y[ts], hn, cn
    errs = {"y": float(np.abs(ys.cpu().double().numpy() - gold["y"][:, :32]).max()),
            "hn": float(np.abs(hs.cpu().double().numpy() - gold["hn"][:, :32]).max()),
            "cn": float(np.abs(cs.cpu().double().numpy() - gold["cn"][:, :32]).max())}
    print(f"c5 B=32 shard: plan {ex.plan()} max-abs {errs}")
    assert max(errs.values()) <= TOL["bf16"], errs


def test_c2_host_request_path_matches_golden(golden_dir):
    """The end-to-end request path (hs_rnn_forward_host: overlapped H2D/D2H,
    request overlap in a stream of two) at c2 full size."""
    from paper_2307_11339_b200.serve import InferenceRequest, RNNServer

    spec = CONFIGS["c2"]
    gold = np.load(golden_dir / "tensor_c2.npz")
    ex = RNNExecutor(spec, init_weights(spec, 0))
    server = RNNServer(ex)
    req = InferenceRequest(x=make_input(spec, 1).pin_memory())
    outs = []
    server.run_stream([req, req, req], consume=lambda i, r: outs.append((r.y.clone(), r.hn.clone(), r.cn.clone())))
    assert len(outs) == 3
    for y, hn, cn in outs:
        errs = compare(gold, y, hn, cn, spec.seq, spec.batch)
        print(f"c2 request path: max-abs {errs}")
        assert max(errs.values()) <= TOL["f32"], errs
