"""The production kernel families at reduced T, for compute-sanitizer runs
(racecheck / synccheck / memcheck): the two-group recurrence at c2 width
(B=64) with the dynamic next-layer K1, the layer-wave fused kernel at c3
width, the W-streaming recurrence at c4 width (H=2048), the batch-sliced bf16
path at c5 width, the host-buffer request stream (request overlap, async
output drain), two layer-pipeline stages (stream-ordered peer hand-off) and
hybrid-plan GPU segments (hs_rnn_run_cells on the small-shape cluster kernel
and on the tensor-core path, reverse direction included)."""
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
    srv.run_stream([InferenceRequest(x=make_input(spec, 1 + i).pin_memory()) for i in range(4)])  # async output drain
    torch.cuda.synchronize()
    print("ok request stream", flush=True)
if not only or "stage" in only:
    # two pipeline stages in one process, producer enqueued first (hs_rnn_forward_stage)
    from paper_2307_11339_b200.parallel import stage_link_values
    from paper_2307_11339_b200.rnn import StageLink

    spec = RNNSpec("lstm", 2, 256, 8, 16, algo="tc")
    w = init_weights(spec)
    e0 = RNNExecutor(spec.with_(layers=1), w[:1])
    e1 = RNNExecutor(spec.with_(layers=1, input=spec.hidden), w[1:])
    T, B, H = spec.seq, spec.batch, spec.hidden
    slots = torch.zeros((2, 2, T * B, H), dtype=torch.bfloat16, device="cuda")
    avail = torch.zeros(1, dtype=torch.int32, device="cuda")
    consumed = torch.zeros(1, dtype=torch.int32, device="cuda")
    for r in range(2):
        v0, v1 = stage_link_values(r, T, 0, 2), stage_link_values(r, T, 1, 2)
        e0.forward_stage(StageLink(y_peer_planes=slots[r % 2].data_ptr(), y_peer_avail=avail.data_ptr(),
                                   y_base=v0["y_base"], consumed=consumed.data_ptr(),
                                   consumed_wait=v0["consumed_wait"], chunks=2), x=make_input(spec, r).cuda())
        e1.forward_stage(StageLink(x_planes=slots[r % 2].data_ptr(), x_avail=avail.data_ptr(), x_base=v1["x_base"],
                                   consumed_peer=consumed.data_ptr(), consumed_value=v1["consumed_value"], chunks=2))
    torch.cuda.synchronize()
    print("ok pipeline stages", flush=True)
if not only or "segments" in only:
    # hybrid-plan GPU segments: three segments per layer-direction
    for spec in (RNNSpec("lstm", 2, 96, 7, 3, input=40, dirs=2, algo="simt"),
                 RNNSpec("gru", 2, 256, 6, 8, dirs=2, algo="tc")):
        ex = RNNExecutor(spec, init_weights(spec))
        x = make_input(spec).cuda()
        T, B, H, D = spec.seq, spec.batch, spec.hidden, spec.dirs
        inp = x
        for l in range(spec.layers):
            out = torch.zeros((T, B, D * H), device="cuda")
            for d in range(D):
                h = torch.zeros((B, H), device="cuda")
                c = torch.zeros((B, H), device="cuda")
                for t0, t1 in ((0, 2), (2, 4), (4, T)):
                    h2, c2 = torch.empty_like(h), torch.empty_like(c)
                    lstm = spec.cell == "lstm"
                    ex.run_cells(l * D + d, t0, t1, inp, out, h, c if lstm else None, h2, c2 if lstm else None)
                    h, c = h2, c2
            inp = out
        torch.cuda.synchronize()
        print("ok segments", spec.cell, ex.algo, flush=True)
