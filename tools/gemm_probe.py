"""K1 GEMM time at c2 (layer-0 input projection), device path (debug)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
spec = hs.CONFIGS[cfg].with_(layers=1)
ex = hs.RNNExecutor(spec, hs.init_weights(spec))
x = hs.make_input(spec).cuda()
outs = ex.alloc_outputs()
g = []
for i in range(10):
    *_, lm = ex.forward(x, out=outs, layer_ms=True)
    g.append(lm[0][0])
print(f"{cfg} layer-0 K1 (+split) {statistics.median(g[3:]):.4f} ms")
