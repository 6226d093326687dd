"""Kernel timeline of one forward (torch.profiler / CUPTI): start, end and
stream of every kernel and memset, relative to the first — shows which K1
work is exposed and where the gaps between layers are.

  python tools/timeline.py [c2|c3|...] [--host]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c2"
spec = hs.CONFIGS[cfg]
ex = hs.RNNExecutor(spec, hs.init_weights(spec))
x = hs.make_input(spec).cuda()
outs = ex.alloc_outputs()
for _ in range(10):  # synchronised, so per-shape controllers (XP streaming head) see each forward's events
    ex.forward(x, out=outs)
    torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    ex.forward(x, out=outs)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  "
          f"{str(getattr(e, 'device_index', ''))} {e.name[:90]}")
