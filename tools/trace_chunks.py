"""Per-chunk operand arrival inside the recurrence's MMA loop (debug).

Needs the HS_TRACE_CHUNKS diagnostic build (the MMA issuer first waits for
every h chunk of the step and records when each landed):
  python -c "from paper_2307_11339_b200 import build as b; \\
             b.build(True, out='paper_2307_11339_b200/_lib/libhsrnn_tc.so', defines=('HS_TRACE_CHUNKS',))"
  HS_LIB_PATH=paper_2307_11339_b200/_lib/libhsrnn_tc.so python tools/trace_chunks.py c4
Prints medians over layer 0's launch, steps 2..60, all CTAs.
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
out = sys.argv[2] if len(sys.argv) > 2 else "/tmp/trace_chunks.bin"
os.environ["HS_RECUR_TRACE"] = out

import torch  # noqa: E402

from paper_2307_11339_b200 import CONFIGS, RNNExecutor, init_weights, make_input  # noqa: E402

spec = CONFIGS[cfg].with_(algo="tc")
ex = RNNExecutor(spec, init_weights(spec))
x = make_input(spec).cuda()
for _ in range(3):
    ex.forward(x)
torch.cuda.synchronize()
tr = np.fromfile(out, dtype=np.uint64).reshape(320, 64, 16).astype(np.int64)
ncta = int((tr[:, :, 0] > 0).any(axis=1).sum())
tr = tr[:ncta, 2:60]
nch = min(int((tr[0, 0, :14] > 0).sum()), 14)
rel = tr[:, :, :nch] - tr[:, :, :1]
if (tr[:, :, 14] > 0).any():
    v = tr[:, :, 14] - tr[:, :, nch - 1]
    print(f"{cfg}: the TMEM-resident chunks' MMAs alone, issued after every h chunk landed: "
          f"median {np.median(v) / 1e3:.2f} us  p90 {np.percentile(v, 90) / 1e3:.2f}")
print(f"{cfg}: {ncta} CTAs; h chunk c landed, relative to chunk 0 (us)")
for c in range(nch):
    print(f"  chunk {c:2d}  median {np.median(rel[:, :, c]) / 1e3:6.2f}  p90 {np.percentile(rel[:, :, c], 90) / 1e3:6.2f}")
per = np.median(tr[:, 1:, 0] - tr[:, :-1, 0]) / 1e3
print(f"  step period (chunk 0 to chunk 0) median {per:.2f} us")
