"""Host-buffer forward (hs_rnn_forward_host / run(request)): chunked H2D of x
overlapped with the layer-0 input projection and chunked D2H of y overlapped
with the last recurrence must give exactly the device-resident forward."""
import pytest
import torch

from paper_2307_11339_b200 import CONFIGS, InferenceRequest, RNNExecutor, RNNSpec, init_weights, make_input, register_model, run

pytestmark = pytest.mark.gpu

SPECS = [
    CONFIGS["c2"].with_(seq=40),                       # tensor-core path, 8 ragged-free chunks
    RNNSpec("gru", 2, 256, 13, 24, dirs=2, algo="tc"),  # bidirectional drain order, ragged chunks
    RNNSpec("lstm", 3, 128, 5, 16, input=64, algo="tc"),  # T < 8 chunks
    RNNSpec("lstm", 2, 48, 9, 3),                      # SIMT path (no overlap)
    CONFIGS["c2"].with_(seq=24, dtype="bf16"),
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"{s.cell}{s.layers}x{s.hidden}T{s.seq}B{s.batch}d{s.dirs}{s.dtype}")
def test_forward_host_equals_device_forward(spec):
    w = init_weights(spec, 1)
    ex = RNNExecutor(spec, w)
    x = make_input(spec, 2).pin_memory()
    gen = torch.Generator().manual_seed(3)
    shp = (spec.layers * spec.dirs, spec.batch, spec.hidden)
    h0 = (torch.rand(shp, generator=gen) - 0.5).pin_memory()
    c0 = (torch.rand(shp, generator=gen) - 0.5).pin_memory() if spec.cell == "lstm" else None
    for states in ((None, None), (h0, c0)):
        dev = ex.device
        ref = ex.forward(x.to(dev), *(None if t is None else t.to(dev) for t in states))
        ref = [t.cpu() if t is not None else None for t in ref]
        for _ in range(2):  # second call re-uses staging/counters
            got = ex.forward_host(x, *states)
            torch.cuda.current_stream(dev).synchronize()
            for g, r in zip(got, ref):
                if r is not None:
                    assert torch.equal(g, r)


def test_run_request_host_path():
    spec = CONFIGS["c2"].with_(seq=16)
    ex = RNNExecutor(spec, init_weights(spec))
    register_model("t", ex)
    x = make_input(spec).pin_memory()
    resp = run(InferenceRequest(x=x, model="t"))
    y, hn, cn = ex.forward(x.to(ex.device))
    assert torch.equal(resp.y, y.cpu()) and torch.equal(resp.hn, hn.cpu()) and torch.equal(resp.cn, cn.cpu())
    assert resp.h2d_bytes == x.numel() * 4 and resp.device_ms > 0


@pytest.mark.parametrize("spec", [
    CONFIGS["c2"].with_(seq=24),
    RNNSpec("gru", 2, 256, 13, 24, dirs=2, algo="tc"),  # bidirectional: both directions' K1 in one dynamic launch
    CONFIGS["c3"].with_(seq=20),                        # 4 layers: xproj ping-pong across requests
    RNNSpec("lstm", 3, 256, 9, 16, algo="tc"),          # odd layer count: no request overlap
], ids=["c2", "gru-bidir", "c3", "lstm-3layer"])
def test_run_stream_pipelined_requests(spec):
    """RNNServer.run_stream: request i+1's upload overlaps request i's compute
    (alternating staging slots) and, for even layer counts, its layer-0 input
    projection overlaps request i's last recurrence; every request's outputs
    must still be exact."""
    from paper_2307_11339_b200 import RNNServer

    ex = RNNExecutor(spec, init_weights(spec, 4))
    xs = [make_input(spec, 10 + i).pin_memory() for i in range(5)]
    refs = [[None if t is None else t.cpu() for t in ex.forward(x.to(ex.device))] for x in xs]
    server = RNNServer(ex)
    got = {}
    server.run_stream([InferenceRequest(x=x) for x in xs], consume=lambda i, r: got.__setitem__(i, tuple(None if t is None else t.clone() for t in (r.y, r.hn, r.cn))))
    assert sorted(got) == list(range(5))
    for i in range(5):
        for g, r in zip(got[i], refs[i]):
            assert (g is None and r is None) or torch.equal(g, r)
