"""e2e request-stream time per request at c2 (debug)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

spec = hs.CONFIGS["c2"]
ex = hs.RNNExecutor(spec, hs.init_weights(spec))
x = hs.make_input(spec).pin_memory()
srv = hs.RNNServer(ex)
req = hs.InferenceRequest(x=x)
srv.run_stream([req] * 3)
r = srv.run_stream([req] * 20)
xd = x.cuda()
outs = ex.alloc_outputs()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ex.forward(xd, out=outs)
e0.record()
for _ in range(20):
    ex.forward(xd, out=outs)
e1.record()
e1.synchronize()
print(f"stream e2e {r.device_ms / 20:.3f} ms/request; device forward back-to-back {e0.elapsed_time(e1) / 20:.3f} ms")
