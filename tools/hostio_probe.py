"""Time the pieces of the host-buffer forward at c2 (debug): H2D of x alone,
D2H of y alone, device forward, and hs_rnn_forward_host end to end."""
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HS_DEBUG", "1")
import torch  # noqa: E402

from paper_2307_11339_b200 import CONFIGS, RNNExecutor, init_weights, make_input  # noqa: E402

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
ex = RNNExecutor(spec, init_weights(spec))
x = make_input(spec).pin_memory()
xd = x.cuda()
outs = ex.alloc_outputs()
hosts = ex.alloc_host_outputs()
stg = ex.alloc_staging()


def timeit(fn, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


print("h2d x      ms", timeit(lambda: xd.copy_(x, non_blocking=True)))
print("d2h y      ms", timeit(lambda: hosts[0].copy_(outs[0], non_blocking=True)))
print("forward    ms", timeit(lambda: ex.forward(xd, out=outs)))
print("fwd_host   ms", timeit(lambda: ex.forward_host(x, out_host=hosts, staging=stg)))
print("sequential ms", timeit(lambda: (xd.copy_(x, non_blocking=True), ex.forward(xd, out=outs),
                                       hosts[0].copy_(outs[0], non_blocking=True))))
