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
tr = np.fromfile(out, dtype=np.uint64).reshape(320, 64, 16).astype(np.int64)
used = tr[:, :, 0] > 0
ncta = int(used.any(axis=1).sum())
tr = tr[:ncta]
S = 4 if cfg == "c2" else int(os.environ.get("TRACE_S", "8"))
H = spec.hidden
KS = H // S
nch = KS // 64
T0, T1 = 2, 60
def med(x):
    return np.median(x) / 1e3
def ph(i):
    return tr[:, T0:T1, i]
print(f"{cfg}: {ncta} CTAs, S={S}, nch={nch}")
rows = [
    ("producer: top -> chunk0 ready", 0, 1),
    ("producer: chunk0 ready -> last ready", 1, 12),
    ("mma: chunk0 landed -> last landed", 15, 14),
    ("mma: last ready -> last landed", 12, 14),
    ("mma: last landed -> commit issued", 14, 2),
    ("epi: commit -> acc_full seen", 2, 3),
    ("epi: tmem ld + dsmem stores", 3, 4),
    ("epi: cluster barrier", 4, 5),
    ("epi: gates + h stores", 5, 6),
    ("epi: fence.proxy + bar.sync", 6, 8),
    ("epi: bar -> release issued", 8, 10),
    ("epi: release -> end (outputs, prefetch)", 10, 11),
]
for name, a_, b_ in rows:
    v = ph(b_) - ph(a_)
    print(f"  {name:42s} median {med(v):6.2f} us  p90 {np.percentile(v, 90)/1e3:6.2f}")
v = tr[:, T0 + 1:T1 + 1, 0] - tr[:, T0:T1, 11]
print(f"  end of step -> next top  median {med(v):.2f} us")
lat = []
for cta in range(ncta):
    q = cta % S
    j0 = (q * KS) // 64
    prods = [rb * S + qq for rb in (2 * j0, 2 * j0 + 1) for qq in range(S)]
    for s_ in range(T0 + 1, T1):
        lat.append(tr[cta, s_, 1] - tr[prods, s_ - 1, 10].max())
print(f"  last producer release -> chunk0 seen  median {med(np.array(lat)):.2f} us")
period = tr[:, T0 + 1:T1 + 1, 10] - tr[:, T0:T1, 10]
print(f"  step period (release to release) median {med(period):.2f} us")
