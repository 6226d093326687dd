"""Regenerate tests/golden/tensor_c1.npz: config c1 (1-layer LSTM H128, T16,
B1) with init_weights(seed=0), make_input(seed=1), outputs from the float64
oracle (oracle/rnn_ref.py).  The reference has no tensor numerics, so this
fixture pins the oracle's own output (parity against the reference unpinned)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle.rnn_ref import rnn_forward_ref  # noqa: E402
from paper_2307_11339_b200 import CONFIGS, init_weights, make_input  # noqa: E402

spec = CONFIGS["c1"]
w = init_weights(spec, 0)
x = make_input(spec, 1)
y, hn, cn = rnn_forward_ref("lstm", x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w])
np.savez_compressed(Path(__file__).with_name("tensor_c1.npz"), x=x.numpy(), y=y, hn=hn, cn=cn)
