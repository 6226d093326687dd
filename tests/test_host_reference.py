"""The host-CPU reference arm (oracle/rnn_cells_f32.py):
fp32 torch, one dispatch per cell in Plan.order, checked against the float64
oracle; plus bench.py's reference-arm plumbing on a small config."""
import importlib.util
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.rnn_cells_f32 import cells_forward_f32, fused_forward_f32, plan_order
from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import RNNSpec, init_weights, make_input

ROOT = Path(__file__).resolve().parents[1]

SPECS = [
    RNNSpec("lstm", 2, 32, 9, 3),
    RNNSpec("gru", 3, 24, 7, 2, input=12),
    RNNSpec("lstm", 2, 16, 6, 4, dirs=2),
    RNNSpec("gru", 2, 20, 5, 3, input=8, dirs=2),
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"{s.cell}{s.layers}x{s.hidden}T{s.seq}d{s.dirs}")
def test_cells_in_plan_order_match_oracle(spec):
    w = init_weights(spec, 0)
    x = make_input(spec, 1)
    order, _src = plan_order(spec)
    assert sorted(order) == list(range(spec.layers * spec.dirs * spec.seq))
    y, hn, cn = cells_forward_f32(spec.cell, x, w, order, dirs=spec.dirs)
    ref = rnn_forward_ref(spec.cell, x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w],
                          dirs=spec.dirs, order=order)
    for g, r in zip((y, hn, cn), ref):
        if r is not None:
            assert float(np.abs(g.double().numpy() - r).max()) <= 1e-5
    fy, st = fused_forward_f32(spec, w)(x)
    fh = st[0] if spec.cell == "lstm" else st
    assert float((fy - y).abs().max()) <= 1e-5
    assert float((fh - hn).abs().max()) <= 1e-5


def test_reference_arm_line():
    """bench.py --impl reference prints one JSON line: fp32 host path, checked
    against the oracle, with the fused path beside it (c1: seconds on CPU)."""
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "2",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["dtype"] == "f32" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["max_abs_vs_f64_oracle"] <= 1e-4
    assert cb["torch_fused_fp32"]["value"] > 0
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
