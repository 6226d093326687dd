"""Per-phase timeline of the tensor-core recurrent kernel (debug).

Runs one config with HS_RECUR_TRACE set (layer 0's recurrent launch records
%globaltimer stamps per CTA per step) and prints median phase durations.
usage: python tools/trace_recur.py [config] [out.bin]
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
out = sys.argv[2] if len(sys.argv) > 2 else str(ROOT / "gpurun_out" / f"trace_{cfg}.bin")
os.environ["HS_RECUR_TRACE"] = out

import torch  # noqa: E402

from paper_2307_11339_b200 import CONFIGS, RNNExecutor, init_weights, make_input  # noqa: E402

spec = CONFIGS[cfg].with_(algo="tc")
ex = RNNExecutor(spec, init_weights(spec))
x = make_input(spec).cuda()
for _ in range(3):
    ex.forward(x)
torch.cuda.synchronize()
tr = np.fromfile(out, dtype=np.uint64).reshape(160, 64, 8).astype(np.int64)
used = tr[:, :, 0] > 0
ncta = int(used.any(axis=1).sum())
tr = tr[:ncta]
names = ["wait_ctr", "h_load+mma_issue", "mma_tail", "scatter", "cluster_bar", "epilogue->release", "tail"]
print(f"{cfg}: {ncta} CTAs")
steps = range(2, 60)
for i, n in enumerate(names):
    a, b = i, i + 1
    dur = np.array([tr[:, s, b] - tr[:, s, a] for s in steps])
    ok = (tr[:, 2:60, a] > 0) & (tr[:, 2:60, b] > 0)
    v = dur.T[ok]
    print(f"  {n:20s} median {np.median(v)/1e3:7.2f} us   p90 {np.percentile(v,90)/1e3:7.2f} us")
period = np.array([tr[:, s + 1, 0] - tr[:, s, 0] for s in steps])
print(f"  step period median {np.median(period)/1e3:.2f} us")
# skew of release times across CTAs per step
rel = tr[:, 2:60, 6]
print(f"  release skew (max-min over CTAs) median {np.median(rel.max(0)-rel.min(0))/1e3:.2f} us")
