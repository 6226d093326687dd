"""Kernel/copy timeline of a host-buffer request stream (RNNServer.run_stream,
the bench's e2e path) via torch.profiler (CUPTI): start, end, duration and
stream of every kernel / memcpy of 4 consecutive requests, relative to the
first — shows what is exposed between consecutive requests' recurrences.

  python tools/timeline_stream.py [c2|...] [nreq]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2307_11339_b200 as hs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = hs.CONFIGS[cfg]
ex = hs.RNNExecutor(spec, hs.init_weights(spec))
srv = hs.RNNServer(ex)
reqs = [hs.InferenceRequest(x=hs.make_input(spec, i).pin_memory()) for i in range(nreq)]
for _ in range(3):
    srv.run_stream(reqs)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    srv.run_stream(reqs)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  "
          f"{getattr(e, 'device_index', 0)} {e.name[:100]}")
