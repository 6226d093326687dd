"""Multi-GPU host logic on CPU: world-size-2 gloo process groups.

Request sharding must reproduce the single-process forward slice for slice.
The layer pipeline (chunked, with point-to-point hand-off) must reproduce the
float64 oracle on the last stage and each stage's final states. The stage
models here are host models; on the B200 box the same code runs RNNExecutor
stages over NCCL peer sends.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import RNNSpec, init_weights, make_input
from paper_2307_11339_b200.parallel import HostStage, LayerPipeline, RequestShard, shard_range, stage_layers

TOL = 1e-4


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle(spec, w, x):
    return rnn_forward_ref(spec.cell, x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w],
                           dirs=spec.dirs)


def test_shard_range_partitions():
    for batch in range(0, 20):
        for world in range(1, 9):
            parts = [shard_range(batch, world, r) for r in range(world)]
            assert sum(c for _, c in parts) == batch
            pos = 0
            for s, c in parts:
                assert s == pos and c >= 0
                pos += c
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
    assert stage_layers(8, 4, 3) == (6, 8)
    with pytest.raises(ValueError):
        stage_layers(2, 4, 0)


def test_request_shards_concatenate_to_full():
    spec = RNNSpec("lstm", 2, 12, 5, 7, dirs=2)
    w = init_weights(spec, 1)
    x = make_input(spec, 2)
    ry, rhn, rcn = oracle(spec, w, x)
    ys, hns, cns = [], [], []
    for rank in range(3):
        sh = RequestShard(spec, lambda sp: _HostFull(sp, w), rank, 3)
        start, y, hn, cn = sh.forward(x)
        assert start == shard_range(7, 3, rank)[0]
        ys.append(y), hns.append(hn), cns.append(cn)
    y = torch.cat(ys, 1).double().numpy()
    assert np.abs(y - ry).max() <= TOL
    assert np.abs(torch.cat(hns, 1).double().numpy() - rhn).max() <= TOL
    assert np.abs(torch.cat(cns, 1).double().numpy() - rcn).max() <= TOL


class _HostFull:
    """Whole-stack host model (any dirs) via the all-host plan executor."""

    def __init__(self, spec, w):
        from paper_2307_11339_b200 import graph, planner
        from paper_2307_11339_b200.executor import HostRNN

        self.spec = spec
        self.host = HostRNN(spec, w)
        g = graph.gen_lstm_grid(spec.layers, spec.seq) if spec.dirs == 1 else graph.gen_bilstm_grid(spec.layers, spec.seq)
        self.g = g
        self.plan = planner.Plan(order=planner.topo_sort_bfs(g), selection=(1,) * g.n, cores=(1,) * g.n,
                                 k_star=1, alpha=0.0)

    def forward(self, x, h0=None, c0=None):
        from paper_2307_11339_b200.executor import execute

        r = execute(self.g, self.plan, self.host, x, h0, c0)
        return r.y, r.hn, r.cn


def _pipeline_worker(rank, world, port, spec, chunk, nreq, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = init_weights(spec, 3)
        xs = [make_input(spec, 10 + r) for r in range(nreq)]
        pipe = LayerPipeline(spec, w, rank, world, chunk, lambda sp, ww: HostStage(sp, ww))
        res = pipe.run_many(xs if rank == 0 else [None] * nreq)
        out = []
        for r, pr in enumerate(res):
            ry, rhn, rcn = oracle(spec, w, xs[r])
            l0, l1 = pipe.l0, pipe.l1
            e = float(np.abs(pr.hn.double().numpy() - rhn[l0:l1]).max())
            if rcn is not None:
                e = max(e, float(np.abs(pr.cn.double().numpy() - rcn[l0:l1]).max()))
            if pr.y is not None:
                e = max(e, float(np.abs(pr.y.double().numpy() - ry).max()))
            out.append((r, pr.y is not None, e))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize(
    "spec,chunk,nreq",
    [
        (RNNSpec("lstm", 4, 16, 10, 3, input=8), 4, 2),   # ragged last chunk, 2 requests in flight
        (RNNSpec("gru", 3, 12, 6, 2), 3, 1),               # uneven layer split (2 + 1)
        (RNNSpec("lstm", 2, 8, 5, 2), 16, 1),              # chunk > T: one chunk
    ],
)
def test_layer_pipeline_gloo_world2(spec, chunk, nreq):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, spec, chunk, nreq, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(got) == [0, 1]
    for rank, out in got.items():
        assert len(out) == nreq
        for r, has_y, e in out:
            assert has_y == (rank == 1)
            assert e <= TOL, f"rank {rank} request {r}: max-abs {e}"


def _shard_worker(rank, world, port, spec, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = init_weights(spec, 4)
        x = make_input(spec, 5)
        sh = RequestShard(spec, lambda sp: _HostFull(sp, w), rank, world)
        start, y, hn, cn = sh.forward(x)
        # gather only to check; the data path itself has no collective
        parts = [None] * world
        dist.all_gather_object(parts, (start, y, hn, cn))
        if rank == 0:
            parts.sort(key=lambda p: p[0])
            ry, rhn, rcn = oracle(spec, w, x)
            yy = torch.cat([p[1] for p in parts], 1).double().numpy()
            e = max(float(np.abs(yy - ry).max()),
                    float(np.abs(torch.cat([p[2] for p in parts], 1).double().numpy() - rhn).max()))
            q.put(e)
    finally:
        dist.destroy_process_group()


def test_request_sharding_gloo_world2():
    spec = RNNSpec("gru", 2, 10, 6, 5, input=6, dirs=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, spec, q)) for r in range(2)]
    for p in procs:
        p.start()
    e = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert e <= TOL


def test_pipeline_rejects_bidirectional():
    spec = RNNSpec("lstm", 2, 8, 4, 2, dirs=2)
    with pytest.raises(ValueError):
        LayerPipeline(spec, init_weights(spec), 0, 2, 2, lambda sp, w: HostStage(sp, w))


@pytest.mark.gpu
@pytest.mark.parametrize("spec,chunk", [
    (RNNSpec("lstm", 2, 1024, 48, 64), 16),        # c2 width, tensor-core stages, ragged-free
    (RNNSpec("gru", 2, 512, 20, 32), 8),           # c3 width, ragged last chunk
])
def test_pipeline_single_stage_gpu(spec, chunk):
    """Chunked stage execution with carried (h, c) on the B200 equals the
    oracle (the per-rank body of the NVLink layer pipeline)."""
    from paper_2307_11339_b200 import RNNExecutor

    w = init_weights(spec, 1)
    x = make_input(spec, 2)
    pipe = LayerPipeline(spec, w, 0, 1, chunk, lambda sp, ww: RNNExecutor(sp, ww))
    res = pipe.run(x.pin_memory())
    ry, rhn, rcn = oracle(spec, w, x)
    e = max(float(np.abs(res.y.cpu().double().numpy() - ry).max()),
            float(np.abs(res.hn.cpu().double().numpy() - rhn).max()))
    if rcn is not None:
        e = max(e, float(np.abs(res.cn.cpu().double().numpy() - rcn).max()))
    assert e <= TOL, f"max-abs {e}"
