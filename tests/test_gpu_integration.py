"""The INTEGRATION.md walkthrough, end to end on the B200: a hetsched user's
flow (grid -> measured profile -> plans -> execute -> trace CSV -> requests)."""
import numpy as np
import pytest
import torch

import paper_2307_11339_b200 as hs
from oracle.rnn_ref import rnn_forward_ref

pytestmark = pytest.mark.gpu


def test_integration_walkthrough():
    spec = hs.RNNSpec("lstm", layers=2, hidden=256, seq=12, batch=16)
    weights = hs.init_weights(spec, seed=0)
    model = hs.RNNExecutor(spec, weights, device="cuda:0")
    x = hs.make_input(spec)
    ref = rnn_forward_ref("lstm", x.double().numpy(), [{k: v.double().numpy() for k, v in w.items()} for w in weights])

    g = hs.gen_lstm_grid(spec.layers, spec.seq)
    cm = hs.profile_ops(g, model, k=2, reps=2)
    plan = hs.latency_optimal_plan(g, cm)
    mem_opt = hs.memory_optimal_alpha(g, cm)
    assert mem_opt.latency <= hs.evaluate(g, cm, hs.baseline_plans(g, cm)[0]).latency + 1e-12
    res = hs.execute(g, plan, model, x)
    csv = hs.trace_to_csv(res.trace)
    assert csv.count("\n") >= g.n
    assert float(np.abs(res.y.cpu().double().numpy() - ref[0]).max()) <= 1e-4

    hs.register_model("walkthrough", model)
    resp = hs.run(hs.InferenceRequest(x=x.pin_memory(), model="walkthrough"))
    assert float(np.abs(resp.y.double().numpy() - ref[0]).max()) <= 1e-4

    server = hs.RNNServer(model)
    seen = []
    summary = server.run_stream([hs.InferenceRequest(x=x.pin_memory())] * 3, consume=lambda i, r: seen.append(i))
    assert seen == [0, 1, 2] and summary.h2d_bytes == 3 * x.numel() * 4
    assert torch.equal(summary.y, resp.y)
