"""The production kernel families at reduced T, for compute-sanitizer runs
(racecheck / synccheck / memcheck): the two-group recurrence at c2 width
(B=64) with the dynamic next-layer K1, the layer-wave fused kernel at c3
width, the W-streaming recurrence at c4 width (H=2048), the batch-sliced bf16
path at c5 width, and the host-buffer request stream (request overlap)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_11339_b200 import InferenceRequest, RNNExecutor, RNNServer, RNNSpec, init_weights, make_input  # noqa: E402

CASES = [
    ("two-group c2 width", RNNSpec("lstm", 2, 1024, 6, 64, algo="tc")),
    ("layer wave c3 width", RNNSpec("gru", 4, 512, 6, 32, algo="tc")),
    ("W-streaming c4 width", RNNSpec("lstm", 1, 2048, 3, 16, algo="tc")),
    ("batch-sliced bf16 c5 width", RNNSpec("lstm", 1, 1024, 3, 256, dirs=2, dtype="bf16", algo="tc")),
]
only = sys.argv[1:] and set(sys.argv[1:])
for name, spec in CASES:
    if only and name.split()[0] not in only:
        continue
    ex = RNNExecutor(spec, init_weights(spec))
    x = make_input(spec)
    ex.forward(x.cuda())
    torch.cuda.synchronize()
    print("ok", name, ex.plan(), flush=True)
if not only or "stream" in only:
    spec = RNNSpec("lstm", 2, 1024, 6, 64, algo="tc")  # even layer count: request overlap on
    srv = RNNServer(RNNExecutor(spec, init_weights(spec)))
    srv.run_stream([InferenceRequest(x=make_input(spec, 1 + i).pin_memory()) for i in range(3)])
    torch.cuda.synchronize()
    print("ok request stream", flush=True)
