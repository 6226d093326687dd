"""Real multi-model residency serving on the B200 (serving.ResidencyServer):
swaps move packed weights for real, reloaded models compute bit-identical
outputs, and the measured run follows the reference's accounting
(servingsim.py:143-237) event for event."""
import pytest
import torch

from paper_2307_11339_b200 import RNNExecutor, RNNSpec, init_weights, make_input
from paper_2307_11339_b200.serving import ResidencyServer, Workload, run_serving

pytestmark = pytest.mark.gpu


def _models():
    specs = {"a": RNNSpec("lstm", 1, 128, 16, 8, algo="tc"), "b": RNNSpec("gru", 2, 256, 16, 16, algo="tc"),
             "c": RNNSpec("lstm", 2, 256, 32, 16, algo="tc")}
    return {k: RNNExecutor(s, init_weights(s, i)) for i, (k, s) in enumerate(specs.items())}


def test_offload_load_round_trip_bit_exact():
    spec = RNNSpec("lstm", 2, 256, 16, 16, algo="tc")
    ex = RNNExecutor(spec, init_weights(spec, 3))
    x = make_input(spec, 4).cuda()
    y0, hn0, cn0 = (t.clone() for t in ex.forward(x))
    ex.offload()
    assert not ex.resident
    with pytest.raises(RuntimeError):
        ex.forward(x)
    ex.load()
    y1, hn1, cn1 = ex.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(hn0, hn1) and torch.equal(cn0, cn1)


@pytest.mark.parametrize("policy", ["lru", "fifo"])
def test_measured_serving_follows_reference_accounting(policy):
    models = _models()
    # capacity for the two largest models but not all three: every third request swaps
    probe = ResidencyServer(models, capacity_mb=1e9, policy=policy)
    fp = sorted(probe.footprint_mb.values())
    cap = fp[1] + fp[2] + 1e-3
    srv = ResidencyServer(models, capacity_mb=cap, policy=policy)
    w = Workload(24, "random", 5)
    res, meas = srv.serve(w)
    assert res.metrics.invocations == 24 and len(meas) == 24
    assert res.metrics.swaps > 0
    # the simulated run over the measured scalars makes the same residency decisions
    entries = srv.entries({k: 1.0 for k in models})
    sim = run_serving(entries, cap, w, 1e9, policy)
    kinds = lambda r: [(e.event, e.model, e.detail if e.event == "load" else "") for e in r.events
                       if e.event in ("load", "evict")]
    assert kinds(res) == kinds(sim)
    for m in meas:
        assert m.exec_ms > 0 and m.latency_ms >= m.exec_ms
    # every measured load moved the model's packed bytes
    loads = [m for m in meas if m.load_ms > 0]
    assert len(loads) == sum(e.event == "load" for e in res.events)
