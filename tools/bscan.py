"""Recurrent step time vs batch at c2 width (debug: how much of a step is batch-proportional)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

for B in (8, 16, 32, 64, 128):
    spec = hs.CONFIGS["c2"].with_(batch=B, layers=1, algo="tc")
    ex = hs.RNNExecutor(spec, hs.init_weights(spec))
    x = hs.make_input(spec).cuda()
    outs = ex.alloc_outputs()
    rec = []
    for i in range(8):
        *_, lm = ex.forward(x, out=outs, layer_ms=True)
        rec.append(lm[0][1])
    print(f"B={B}: recurrence {statistics.median(rec[2:]):.3f} ms, {1e3 * statistics.median(rec[2:]) / spec.seq:.2f} us/step")
