"""K1 pass schemes of the f32 mode (tc_gemm.cuh, hs_rnn.cu k1_scheme).

Layer 0 projects the raw input with three bf16 products; the hidden layers
project h with two fp16 products (h rounded to fp16 once, fp16 hi/lo of the
row-scaled W_ih).  Both schemes, and the A/B switch HS_K1_F16_HIDDEN=0
(three products everywhere, run in a subprocess since the library reads the
switch once), stay within the f32 budget of the float64 oracle (max-abs
<= 1e-4, north_star) on multi-layer shapes of every K1 path: the layer-by-
layer schedule with XP streaming, the layer wave, bidirectional layers and
a GRU whose hidden states reach larger magnitudes."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import RNNExecutor, RNNSpec, init_weights, make_input

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
TOL = 1e-4

SPECS = [
    RNNSpec("lstm", 3, 1024, 24, 64, algo="tc"),           # c2 width, XP streaming
    RNNSpec("gru", 4, 512, 32, 32, algo="tc"),             # c3 width, layer wave
    RNNSpec("lstm", 2, 512, 12, 32, dirs=2, algo="tc"),    # bidirectional hidden layer (K = 2H)
]
IDS = [f"{s.cell}{s.layers}x{s.hidden}T{s.seq}B{s.batch}d{s.dirs}" for s in SPECS]


def _errs(spec, outs):
    w = init_weights(spec, 7)
    x = make_input(spec, 8)
    ry, rhn, rcn = rnn_forward_ref(spec.cell, x.double().numpy(),
                                   [{k: v.double().numpy() for k, v in d.items()} for d in w], dirs=spec.dirs)
    e = {"y": float(np.abs(outs[0] - ry).max()), "hn": float(np.abs(outs[1] - rhn).max())}
    if rcn is not None:
        e["cn"] = float(np.abs(outs[2] - rcn).max())
    return e


def _run(spec):
    ex = RNNExecutor(spec, init_weights(spec, 7))
    y, hn, cn = ex.forward(make_input(spec, 8).cuda())
    torch.cuda.synchronize()
    return [t.cpu().double().numpy() if t is not None else None for t in (y, hn, cn)]


@pytest.mark.parametrize("spec", SPECS, ids=IDS)
def test_hidden_layer_fp16_k1_within_budget(spec):
    errs = _errs(spec, _run(spec))
    print(f"{spec.cell} {spec.layers}x{spec.hidden} d{spec.dirs}: max-abs {errs}")
    assert max(errs.values()) <= TOL, errs


@pytest.mark.parametrize("spec", SPECS[:2], ids=IDS[:2])
def test_three_product_k1_everywhere_within_budget(spec, tmp_path):
    """HS_K1_F16_HIDDEN=0: every layer on the three-product scheme (subprocess)."""
    out = tmp_path / "out.npz"
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, '.');"
        "from paper_2307_11339_b200 import RNNExecutor, RNNSpec, init_weights, make_input;"
        f"s = RNNSpec({spec.cell!r}, {spec.layers}, {spec.hidden}, {spec.seq}, {spec.batch}, dirs={spec.dirs}, algo='tc');"
        "ex = RNNExecutor(s, init_weights(s, 7)); y, hn, cn = ex.forward(make_input(s, 8).cuda()); torch.cuda.synchronize();"
        f"np.savez({str(out)!r}, y=y.cpu().double().numpy(), hn=hn.cpu().double().numpy(),"
        " cn=(cn.cpu().double().numpy() if cn is not None else np.zeros(0)))"
    )
    env = dict(os.environ, HS_K1_F16_HIDDEN="0")
    p = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    z = np.load(out)
    outs = [z["y"], z["hn"], z["cn"] if z["cn"].size else None]
    errs = _errs(spec, outs)
    assert max(errs.values()) <= TOL, errs
    # and the two schemes agree with each other within the same budget
    cur = _run(spec)
    assert float(np.abs(cur[0] - outs[0]).max()) <= TOL
