"""Kernel/copy timeline of one single-request host forward (forward_host,
pinned x in, y/h_n/c_n out) via torch.profiler (CUPTI).

  python tools/timeline_host.py [c2|...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
spec = hs.CONFIGS[cfg]
ex = hs.RNNExecutor(spec, hs.init_weights(spec))
x = hs.make_input(spec).pin_memory()
for _ in range(8):
    ex.forward_host(x)
    torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    ex.forward_host(x)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:80]}")
