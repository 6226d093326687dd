"""Multi-GPU modes of the RNN DAG forward: one process per GPU.

The path shards two ways, and neither needs a collective:

* **Request sharding** (:func:`shard_range`, :class:`RequestShard`): sequences
  are independent, so the batch of a request (or a stream of requests) is
  split across ranks. Weights are replicated and each rank computes and
  returns its own slice. The data path has no communication. This is the
  scaling mode for c2/c5 and for ``bench.py --gpus N``.
* **Layer pipeline** (:class:`LayerPipeline`): rank g owns the contiguous
  layer range ``stage_layers(L, N, g)`` and runs it over time chunks of
  ``chunk`` steps. It carries (h, c) from chunk to chunk and passes each
  chunk's output ``[chunk, B, H]`` to rank g+1 with a point-to-point send.
  Under NCCL on an NVSwitch box that send is an NVLink peer copy. Rank g's
  chunk k therefore overlaps rank g+1's chunk k−1: this is the layer
  wavefront (layer l step t ‖ layer l+1 step t−1) at chunk granularity and
  across GPUs. There is one exchange per chunk per stage boundary and no
  allreduce. Bidirectional stacks cannot be pipelined over time, because
  layer l+1 at t needs layer l's backward output at t, which is produced
  last. Those stacks use request sharding.

  With ``handoff="peer"`` (:class:`PeerPipeline`) each stage instead runs
  the whole sequence in ONE stage forward (``hs_rnn_forward_stage``): its last
  layer's output planes are copied GPU-to-GPU by the copy engine into the
  next stage's input slot, chunk by chunk as the recurrence publishes steps,
  and the next stage's input projection consumes each chunk as it lands.
  Synchronisation is stream-ordered on monotonic 32-bit counters in GPU
  memory (cuStreamWaitValue32 / cuStreamWriteValue32), shared between the
  processes by CUDA IPC; no kernel spins on another GPU and there is no NCCL
  call on the data path. No relaunch per chunk, no W_hh reload.

The reference has no multi-device execution: its "devices" are virtual
processors inside one process (costmodel.py:3-11, engine.py:37; SPEC.md:451
lists multi-GPU clusters as a non-goal). Plans carry no GPU index, so these
modes map a plan's GPU cells onto devices by request or by layer. That keeps
plan bit-exactness intact.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .rnn import RNNSpec

__all__ = ["shard_range", "stage_layers", "RequestShard", "LayerPipeline", "HostStage", "PeerPipeline",
           "stage_link_values"]


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous split of ``batch`` sequences over ``world`` ranks.

    Returns ``(start, count)``. The first ``batch % world`` ranks get one
    extra sequence, so a rank may get zero sequences when ``batch < world``.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if batch < 0:
        raise ValueError("batch must be non-negative")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def stage_layers(layers: int, world: int, rank: int) -> tuple[int, int]:
    """Layer range ``[l0, l1)`` owned by pipeline stage ``rank``."""
    if layers < world:
        raise ValueError(f"cannot pipeline {layers} layers over {world} stages")
    s, c = shard_range(layers, world, rank)
    return s, s + c


class RequestShard:
    """This rank's slice of every request, run on its own executor.

    ``make_executor(spec)`` builds the per-rank model. It is an
    :class:`~paper_2307_11339_b200.rnn.RNNExecutor` on the rank's GPU; tests
    pass a host model. :meth:`forward` takes the full request and returns
    this rank's ``(start, y, h_n, c_n)``. The outputs are not gathered over
    the network: the caller owns the slices, and concatenating them along the
    batch axis is the full result.
    """

    def __init__(self, spec: RNNSpec, make_executor, rank: int, world: int):
        self.spec = spec
        self.rank, self.world = rank, world
        self.start, self.count = shard_range(spec.batch, world, rank)
        self.local_spec = spec.with_(batch=max(self.count, 1))
        self.model = make_executor(self.local_spec) if self.count else None

    def forward(self, x, h0=None, c0=None):
        if self.count == 0:
            return self.start, None, None, None
        sl = slice(self.start, self.start + self.count)
        xs = x[:, sl].contiguous()
        h0s = h0[:, sl].contiguous() if h0 is not None else None
        c0s = c0[:, sl].contiguous() if c0 is not None else None
        dev = getattr(self.model, "device", None)
        if dev is not None and dev.type == "cuda":
            xs = xs.to(dev, non_blocking=True)
            h0s = h0s.to(dev) if h0s is not None else None
            c0s = c0s.to(dev) if c0s is not None else None
        y, hn, cn = self.model.forward(xs, h0s, c0s)
        return self.start, y, hn, cn


class HostStage:
    """Host-core stage model with the RNNExecutor ``forward`` signature (CPU
    tests of the pipeline logic, and all-host pipelines)."""

    def __init__(self, spec: RNNSpec, weights):
        from .executor import HostRNN

        self.spec = spec
        self.host = HostRNN(spec, weights)
        self.device = torch.device("cpu")

    def forward(self, x, h0=None, c0=None, out=None):
        s = self.spec
        L, T, B, H = s.layers, s.seq, x.shape[1], s.hidden
        lstm = s.cell == "lstm"
        hn = torch.empty((L, B, H))
        cn = torch.empty((L, B, H)) if lstm else None
        inp = x
        for l in range(L):
            h = h0[l] if h0 is not None else torch.zeros(B, H)
            c = (c0[l] if c0 is not None else torch.zeros(B, H)) if lstm else None
            out_l = torch.empty((T, B, H))
            for t in range(T):
                h, c = self.host.cell(l, inp[t], h, c)
                out_l[t] = h
            hn[l] = h
            if lstm:
                cn[l] = c
            inp = out_l
        if out is not None:
            out[0].copy_(inp)
            out[1].copy_(hn)
            if lstm:
                out[2].copy_(cn)
            return out
        return inp, hn, cn


@dataclass
class PipelineResult:
    y: torch.Tensor | None   # [T, B, H] on the last stage, else None
    hn: torch.Tensor         # [layers of this stage, B, H]
    cn: torch.Tensor | None


class LayerPipeline:
    """Stage ``rank`` of a layer pipeline over ``world`` ranks.

    ``make_stage(stage_spec, stage_weights)`` builds the stage model, which
    takes ``forward(x, h0, c0, out=...)``: an RNNExecutor on the rank's GPU,
    or a :class:`HostStage`. The stage spec has ``seq=chunk``, the stage's
    layer count, and input width ``I`` on stage 0 and ``H`` elsewhere.
    A ragged last chunk gets its own stage model.
    """

    def __init__(self, spec: RNNSpec, weights, rank: int, world: int, chunk: int, make_stage, group=None):
        if spec.dirs != 1:
            raise ValueError("bidirectional stacks cannot be layer-pipelined over time; use request sharding")
        if chunk < 1:
            raise ValueError("chunk must be positive")
        self.spec, self.rank, self.world, self.group = spec, rank, world, group
        self.l0, self.l1 = stage_layers(spec.layers, world, rank)
        self.chunk = min(chunk, spec.seq)
        nl = self.l1 - self.l0
        inp = spec.I if rank == 0 else spec.hidden
        self.stage_spec = spec.with_(layers=nl, seq=self.chunk, input=inp)
        w = weights[self.l0:self.l1]
        self.model = make_stage(self.stage_spec, w)
        rem = spec.seq % self.chunk
        self.tail = make_stage(self.stage_spec.with_(seq=rem), w) if rem else None
        self.device = getattr(self.model, "device", torch.device("cpu"))

    @property
    def n_chunks(self) -> int:
        return -(-self.spec.seq // self.chunk)

    def _bounds(self, k):
        t0 = k * self.chunk
        return t0, min(t0 + self.chunk, self.spec.seq)

    def run(self, x=None, h0=None, c0=None) -> PipelineResult:
        """One request through the pipeline.

        Stage 0 needs ``x`` ``[T, B, I]``. ``h0``/``c0``, if given, are the
        stage's own ``[layers of stage, B, H]`` initial states. Returns ``y``
        on the last stage and this stage's final states everywhere.
        """
        return self.run_many([x] if self.rank == 0 else [None], [h0], [c0])[0]

    def run_many(self, xs, h0s=None, c0s=None) -> list[PipelineResult]:
        """A stream of requests, pipelined chunk by chunk. Stage g works on
        (request r, chunk k) while stage g+1 works on the item before it."""
        s = self.spec
        dev = self.device
        B, H = s.batch, s.hidden
        lstm = s.cell == "lstm"
        nl = self.l1 - self.l0
        last = self.rank == self.world - 1
        nreq = len(xs)
        h0s = h0s or [None] * nreq
        c0s = c0s or [None] * nreq
        items = [(r, k) for r in range(nreq) for k in range(self.n_chunks)]
        # double-buffered receive and state buffers
        rbuf = [torch.empty((self.chunk, B, H), device=dev) for _ in range(2)]
        ybuf = [torch.empty((self.chunk, B, H), device=dev) for _ in range(2)]
        st = [(torch.empty((nl, B, H), device=dev), torch.empty((nl, B, H), device=dev) if lstm else None)
              for _ in range(2)]
        results: list[PipelineResult] = []
        pending_recv = None
        pending_send = [None, None]

        def post_recv(i):
            r, k = items[i]
            t0, t1 = self._bounds(k)
            buf = rbuf[i % 2][: t1 - t0]
            return buf, dist.irecv(buf, src=self.rank - 1, group=self.group)

        if self.rank > 0 and items:
            pending_recv = post_recv(0)
        y_full = None
        h, c = None, None
        for i, (r, k) in enumerate(items):
            t0, t1 = self._bounds(k)
            n = t1 - t0
            if k == 0:
                h = h0s[r].to(dev) if h0s[r] is not None else None
                c = c0s[r].to(dev) if (lstm and c0s[r] is not None) else None
                if last:
                    y_full = torch.empty((s.seq, B, H), device=dev)
            if self.rank == 0:
                xin = xs[r][t0:t1].to(dev, non_blocking=True).contiguous()
            else:
                buf, work = pending_recv
                work.wait()
                xin = buf
                if i + 1 < len(items):
                    pending_recv = post_recv(i + 1)
            model = self.model if n == self.chunk else self.tail
            if pending_send[i % 2] is not None:
                pending_send[i % 2].wait()  # ybuf slot free again
                pending_send[i % 2] = None
            y = ybuf[i % 2][:n]
            hs, cs = st[i % 2]
            model.forward(xin, h, c, out=(y, hs, cs))
            h, c = hs, cs
            if not last:
                pending_send[i % 2] = dist.isend(y, dst=self.rank + 1, group=self.group)
            else:
                y_full[t0:t1].copy_(y)
            if k == self.n_chunks - 1:
                results.append(PipelineResult(y_full if last else None, h.clone(), c.clone() if lstm else None))
        for w in pending_send:
            if w is not None:
                w.wait()
        return results


# ------------------------------------------------------- peer (K4) hand-off

def stage_link_values(r: int, T: int, rank: int, world: int) -> dict:
    """Counter values of global request ``r`` on stage ``rank`` (monotonic, so
    they are never reset; include/hs_rnn.h ``hs_stage_link``):

    * input: the slot is ``r % 2``; x_avail reaches ``x_base + T`` when the
      whole request has landed; after reading it the stage sets the previous
      stage's ``consumed`` word to ``r + 1``;
    * output: before the first copy into the next stage's slot ``r % 2`` the
      stage waits for ``consumed >= r - 1`` (request ``r - 2``, the slot's
      previous occupant, has been read).
    """
    v = {"slot": r % 2}
    if rank > 0:
        v.update(x_base=r * T, consumed_value=r + 1)
    if rank < world - 1:
        v.update(y_base=r * T, consumed_wait=max(0, r - 1))
    return v


def _share(t: torch.Tensor):
    from torch.multiprocessing.reductions import reduce_tensor

    return reduce_tensor(t)


def _open(shared):
    fn, args = shared
    return fn(*args)


def _hs_export(lib, t: torch.Tensor):
    """(64-byte CUDA IPC handle, offset) of a device tensor (hs_pipeline_export)."""
    import ctypes

    from .rnn import _check

    h = (ctypes.c_char * 64)()
    off = ctypes.c_size_t()
    _check(lib, "hs_pipeline_export", lib.hs_pipeline_export(t.data_ptr(), h, ctypes.byref(off)))
    return bytes(h), int(off.value)


def _hs_import(lib, exported) -> int:
    """Device address of a peer's exported tensor in this process (hs_pipeline_import)."""
    import ctypes

    from .rnn import _check

    handle, off = exported
    h = (ctypes.c_char * 64).from_buffer_copy(handle)
    p = ctypes.c_void_p()
    _check(lib, "hs_pipeline_import", lib.hs_pipeline_import(h, off, ctypes.byref(p)))
    return int(p.value)


def _addr(x) -> int:
    return x if isinstance(x, int) else x.data_ptr()


class PeerPipeline:
    """Stage ``rank`` of a layer pipeline with the stream-ordered peer hand-off.

    ``executor`` is this stage's :class:`~.rnn.RNNExecutor` (its spec has the
    stage's layers, the full sequence and input width ``I`` on stage 0, ``H``
    elsewhere).  Buffers shared with the neighbours over CUDA IPC:

    * consumer side (rank > 0): two input slots of bf16 hi/lo planes
      ``[2][2][T*B][I]`` and the ``x_avail`` word;
    * producer side (rank < world-1): the ``consumed`` word.

    ``group`` is the process group used once, at construction, to exchange
    the IPC handles (any backend; gloo works for same-host ranks).
    """

    def __init__(self, executor, rank: int, world: int, chunk: int = 32, group=None, share: str = "torch"):
        """``share``: how the link buffers cross processes — "torch"
        (torch.multiprocessing's CUDA tensor sharing) or "hs" (the library's
        own ``hs_pipeline_export`` / ``hs_pipeline_import`` C ABI)."""
        from .rnn import StageLink

        self.ex, self.rank, self.world = executor, rank, world
        s = executor.spec
        if s.dirs != 1:
            raise ValueError("bidirectional stacks cannot be layer-pipelined over time; use request sharding")
        self.T, self.B = s.seq, s.batch
        self.chunks = max(1, -(-s.seq // max(1, chunk)))
        dev = executor.device
        self._StageLink = StageLink
        self.slots = self.x_avail = self.consumed = None
        if rank > 0:
            self.slots = torch.zeros((2, 2, s.seq * s.batch, s.I), dtype=torch.bfloat16, device=dev)
            self.x_avail = torch.zeros(1, dtype=torch.int32, device=dev)
        if rank < world - 1:
            self.consumed = torch.zeros(1, dtype=torch.int32, device=dev)
        if share not in ("torch", "hs"):
            raise ValueError(f"unknown share mode {share!r}")
        self.share = share
        exp = _share if share == "torch" else (lambda t: _hs_export(executor.lib, t))
        mine = {k: exp(t) if t is not None else None
                for k, t in (("slots", self.slots), ("x_avail", self.x_avail), ("consumed", self.consumed))}
        torch.cuda.synchronize(dev)
        allv = [mine]
        if world > 1:
            allv = [None] * world
            dist.all_gather_object(allv, mine, group=group)
        imp = _open if share == "torch" else (lambda h: _hs_import(executor.lib, h))
        self.next_slots = self.next_avail = self.prev_consumed = None
        if rank < world - 1:
            nxt = allv[rank + 1]
            self.next_slots = imp(nxt["slots"])
            self.next_avail = imp(nxt["x_avail"])
        if rank > 0:
            self.prev_consumed = imp(allv[rank - 1]["consumed"])
        self._keep = allv
        self.seq = 0  # global request counter (the monotonic counters' base)

    def link(self, r: int):
        v = stage_link_values(r, self.T, self.rank, self.world)
        lk = self._StageLink()
        lk.chunks = self.chunks
        if self.rank > 0:
            lk.x_planes = self.slots[v["slot"]].data_ptr()
            lk.x_avail = self.x_avail.data_ptr()
            lk.x_base = v["x_base"]
            lk.consumed_peer = _addr(self.prev_consumed)
            lk.consumed_value = v["consumed_value"]
        if self.rank < self.world - 1:
            if self.share == "hs":  # a raw address: slots of the next stage are [2][2][T*B][H] bf16
                lk.y_peer_planes = self.next_slots + v["slot"] * (2 * self.T * self.B * self.ex.spec.hidden * 2)
            else:
                lk.y_peer_planes = self.next_slots[v["slot"]].data_ptr()
            lk.y_peer_avail = _addr(self.next_avail)
            lk.y_base = v["y_base"]
            lk.consumed = self.consumed.data_ptr()
            lk.consumed_wait = v["consumed_wait"]
        return lk

    def run_many(self, xs, h0s=None, c0s=None) -> list[PipelineResult]:
        """A stream of requests.  Stage 0 needs ``xs`` (device or host
        ``[T, B, I]``); other stages pass a list of ``None`` of the same
        length.  Returns ``y`` on the last stage and this stage's final
        states everywhere (copies; all work ordered on the current stream)."""
        ex = self.ex
        n = len(xs)
        h0s = h0s or [None] * n
        c0s = c0s or [None] * n
        outs = []
        for i in range(n):
            r = self.seq + i
            x = xs[i].to(ex.device, torch.float32).contiguous() if self.rank == 0 else None
            y, hn, cn = ex.forward_stage(self.link(r), x=x, h0=h0s[i], c0=c0s[i])
            outs.append(PipelineResult(y if self.rank == self.world - 1 else None, hn, cn))
        self.seq += n
        return outs

    def run(self, x=None, h0=None, c0=None) -> PipelineResult:
        return self.run_many([x], [h0], [c0])[0]
