"""Per-layer timeline of the single-GPU layer wave (debug).

Runs a config with HS_RECUR_TRACE set: every recurrence CTA of the fused wave
records %globaltimer stamps for its first 64 steps.  Prints per layer the
start offset against layer 0, the median step period and the median wait for
the next step's input projection (XP readiness, phases 7 -> 9).
usage: python tools/trace_wave.py [config] [T]
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
out = str(ROOT / "gpurun_out" / f"trace_wave_{cfg}.bin")
os.environ["HS_RECUR_TRACE"] = out

import torch  # noqa: E402

from paper_2307_11339_b200 import CONFIGS, RNNExecutor, init_weights, make_input  # noqa: E402

spec = CONFIGS[cfg].with_(algo="tc")
if len(sys.argv) > 2:
    spec = spec.with_(seq=int(sys.argv[2]))
ex = RNNExecutor(spec, init_weights(spec))
plan = ex.plan()
assert plan["layer_wave"], plan
x = make_input(spec).cuda()
for _ in range(3):
    ex.forward(x)
torch.cuda.synchronize()
tr = np.fromfile(out, dtype=np.uint64).reshape(320, 64, 16).astype(np.int64)
S, L, RB = plan["cluster"], spec.layers, spec.hidden // 32
per = RB * S
t0 = tr[:per, 0, 0].min()
print(f"{cfg} wave: L={L} RB={RB} S={S} ({L * per} recurrence CTAs)")
for l in range(L):
    c = tr[l * per:(l + 1) * per]
    start = (np.median(c[:, 0, 10]) - t0) / 1e3
    period = np.median(c[:, 2:63, 10] - c[:, 1:62, 10]) / 1e3
    xw = c[:, 1:62, 9] - c[:, 1:62, 7]
    prod = np.median(c[:, 2:62, 1] - c[:, 2:62, 0]) / 1e3
    print(f"  layer {l}: step0 release at {start:8.2f} us  period {period:5.2f} us  "
          f"XP wait median {np.median(xw) / 1e3:5.2f} p90 {np.percentile(xw, 90) / 1e3:5.2f} us  "
          f"h-chunk0 wait {prod:5.2f} us")

rows = [
    ("producer: top -> chunk0 ready", 0, 1),
    ("producer: chunk0 ready -> last ready", 1, 12),
    ("producer: last ready -> its TMA issued", 12, 13),
    ("mma: last TMA issued -> last landed", 13, 14),
    ("mma: last landed -> commit issued", 14, 2),
    ("epi: commit -> acc_full seen", 2, 3),
    ("epi: tmem ld + partial staging", 3, 4),
    ("epi: wait partials (red_full)", 4, 5),
    ("epi: gates + h stores", 5, 6),
    ("epi: fence.proxy + bar.sync", 6, 8),
    ("epi: bar -> release issued", 8, 10),
    ("epi: release -> end (outputs, prefetch)", 10, 11),
]
for l in sorted({0, L - 1}):
    c = tr[l * per:(l + 1) * per, 2:62]
    print(f"  layer {l} phases (median over CTAs, steps 2..61):")
    for name, a_, b_ in rows:
        v = c[:, :, b_] - c[:, :, a_]
        print(f"    {name:42s} {np.median(v) / 1e3:6.2f} us  p90 {np.percentile(v, 90) / 1e3:6.2f}")
    v = tr[l * per:(l + 1) * per, 3:63, 0] - tr[l * per:(l + 1) * per, 2:62, 11]
    print(f"    {'end of step -> next top':42s} {np.median(v) / 1e3:6.2f} us")
