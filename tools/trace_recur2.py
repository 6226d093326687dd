"""Per-phase timeline of the two-group recurrent kernel (group 0), debug."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
out = str(ROOT / "gpurun_out" / "trace2.bin")
os.environ["HS_RECUR_TRACE"] = out
import torch  # noqa: E402

from paper_2307_11339_b200 import CONFIGS, RNNExecutor, init_weights, make_input  # noqa: E402

spec = CONFIGS["c2"].with_(algo="tc")
ex = RNNExecutor(spec, init_weights(spec))
x = make_input(spec).cuda()
for _ in range(3):
    ex.forward(x)
torch.cuda.synchronize()
tr = np.fromfile(out, dtype=np.uint64).reshape(320, 64, 16).astype(np.int64)[:128]
T0, T1 = 2, 60
ph = lambda i: tr[:, T0:T1, i]
med = lambda v: np.median(v) / 1e3
for name, a_, b_ in [("top -> chunk0 seen", 0, 1), ("chunk0 -> last chunk seen", 1, 12),
                     ("last seen -> chunk0 landed (MMA thr)", 12, 14), ("chunk0 -> last chunk landed", 14, 15),
                     ("last landed -> commit issued", 15, 2),
                     ("commit -> acc seen (thr 64)", 2, 3), ("red_free wait", 3, 7), ("tmem ld + dsmem stores", 7, 8),
                     ("fence + arrives", 8, 4),
                     ("wait red_full", 4, 5), ("gates + h stores", 5, 6), ("-> release done", 6, 10)]:
    v = ph(b_) - ph(a_)
    print(f"  {name:34s} median {med(v):6.2f} us  p90 {np.percentile(v, 90)/1e3:6.2f}")
period = tr[:, T0 + 1:T1 + 1, 10] - tr[:, T0:T1, 10]
print(f"  step period median {med(period):.2f} us")
