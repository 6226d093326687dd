"""Regenerate the tensor goldens under tests/golden/ (offline, CPU, minutes).

tensor_c1.npz: config c1 (1-layer LSTM H128, T16, B1) in full: x, y, h_n, c_n.
tensor_c2.npz .. tensor_c5.npz: the BASELINE configs at full size (c4: 8x2048
T512 B16; c5: bidirectional 3x1024 T1024 B256), sampled as tensor_sample.py
says, stored as float32 (rounding 6e-8, far below the 1e-4 / 1e-2 budgets).

Inputs are the bench's: init_weights(spec, seed=0), make_input(spec, seed=1)
(CPU torch generators, deterministic).  Outputs come from the float64 oracle
(oracle/rnn_ref.py), evaluated cell by cell in layer-major order.  The
reference has no tensor numerics, so these fixtures pin the oracle's own
output (tensor parity against the reference itself is unpinned).

  python tests/golden/make_tensor_golden.py [c1 c2 ...]
"""
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE))
from oracle.rnn_ref import rnn_forward_ref  # noqa: E402
from paper_2307_11339_b200 import CONFIGS, init_weights, make_input  # noqa: E402
from tensor_sample import sample_index, take  # noqa: E402


def oracle(spec):
    w = init_weights(spec, 0)
    x = make_input(spec, 1)
    y, hn, cn = rnn_forward_ref(spec.cell, x.double().numpy(),
                                [{k: v.double().numpy() for k, v in d.items()} for d in w], dirs=spec.dirs)
    return x, y, hn, cn


def main(names):
    for name in names:
        spec = CONFIGS[name]
        t0 = time.perf_counter()
        x, y, hn, cn = oracle(spec)
        dt = time.perf_counter() - t0
        out = HERE / f"tensor_{name}.npz"
        if name == "c1":
            np.savez_compressed(out, x=x.numpy(), y=y, hn=hn, cn=cn)
        else:
            ys, hs, cs = take(y, hn, cn, spec.seq, spec.batch)
            ts, bs = sample_index(spec.seq, spec.batch)
            arrs = dict(y=ys.astype(np.float32), hn=hs.astype(np.float32), ts=np.array(ts), bs=np.array(bs),
                        oracle_seconds=np.array(dt))
            if cs is not None:
                arrs["cn"] = cs.astype(np.float32)
            np.savez_compressed(out, **arrs)
        print(f"{name}: oracle {dt:.1f} s -> {out.name} ({out.stat().st_size / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
