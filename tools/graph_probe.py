"""Graph replay vs eager forward (RNNExecutor.graph): device time per forward
(CUDA events, 20 back-to-back calls) and host time per call, for the BASELINE
shapes and a few launch-bound ones.  usage: python tools/graph_probe.py [out.json]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_11339_b200 import CONFIGS, RNNExecutor, RNNSpec, init_weights, make_input  # noqa: E402


def timed(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    host = (time.perf_counter() - t0) / n * 1e3
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, host


rows = []
cases = [("c1", CONFIGS["c1"]), ("lstm 2x256 T8 B16", RNNSpec("lstm", 2, 256, 8, 16, algo="tc")),
         ("serving-size lstm 4x256 T32 B1", RNNSpec("lstm", 4, 256, 32, 1, algo="tc")),
         ("gru-bi 2x128 T6 B8", RNNSpec("gru", 2, 128, 6, 8, dirs=2, algo="tc")),
         ("c2", CONFIGS["c2"]), ("c3", CONFIGS["c3"])]
for name, spec in cases:
    ex = RNNExecutor(spec, init_weights(spec))
    x = make_input(spec, 0).cuda()
    out = ex.alloc_outputs()
    gf = ex.graph()
    gf.x.copy_(x)
    dev_e, host_e = timed(lambda: ex.forward(x, out=out))
    dev_g, host_g = timed(lambda: gf.replay())
    r = {"case": name, "spec": str(spec), "eager_ms": round(dev_e, 4), "graph_ms": round(dev_g, 4),
         "eager_host_ms_per_call": round(host_e, 4), "graph_host_ms_per_call": round(host_g, 4)}
    rows.append(r)
    print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(rows, indent=1) + "\n")
