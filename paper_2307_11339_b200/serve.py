"""``run(request)``: the user-facing request path on the B200 executor.

The reference only *simulates* serving (servingsim.run_serving,
/root/reference/pkg/src/hetsched/servingsim.py:143-237, consuming scalar
per-model latencies); a request there is an arrival time and a model name.
Here a request carries real tensors: host (pinned) inputs are copied to the
device, the model's DAG runs on the sm_100a kernels, and outputs are copied
back — all on one CUDA stream, timed with CUDA events so the measured latency
can be fed back into the cost model / serving simulator.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import torch

from .rnn import RNNExecutor

__all__ = ["InferenceRequest", "InferenceResponse", "RNNServer", "register_model", "run"]

# request streams drain each request's outputs off the compute stream
# (hs_rnn_desc.async_outputs); HS_ASYNC_OUT=0 joins them in (A/B)
_ASYNC_OUT = os.environ.get("HS_ASYNC_OUT", "1") != "0"


@dataclass
class InferenceRequest:
    x: torch.Tensor                      # [T, B, I] host (pinned preferred) or device tensor
    h0: torch.Tensor | None = None       # [layers*dirs, B, H]
    c0: torch.Tensor | None = None
    model: str = "default"


@dataclass
class InferenceResponse:
    y: torch.Tensor
    hn: torch.Tensor
    cn: torch.Tensor | None
    device_ms: float                     # H2D + forward + D2H, CUDA events
    h2d_bytes: int
    d2h_bytes: int
    extra: dict = field(default_factory=dict)


class RNNServer:
    """Serves requests for one resident model.

    Device staging and pinned host outputs are preallocated in ``slots``
    sets (default 3), so the request path allocates nothing.  Host requests go through
    ``hs_rnn_forward_host``: within a request, the H2D upload of x and the
    D2H download of y overlap the compute.  :meth:`run_stream` also overlaps
    requests with each other: request i+1's upload runs during request i's
    compute (alternating staging slots; the library makes an upload wait only
    for the previous forward that used the same staging buffer).
    """

    def __init__(self, executor: RNNExecutor, slots: int = 3):
        self.ex = executor
        self.slots = max(1, slots)
        self.staging = [executor.alloc_staging() for _ in range(self.slots)]
        self.host_outs = [executor.alloc_host_outputs() for _ in range(self.slots)]
        self.outs = self.staging[0][1]
        self.ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        self._next = 0

    def _check(self, req: InferenceRequest):
        s = self.ex.spec
        if tuple(req.x.shape) != (s.seq, s.batch, s.I):
            raise ValueError(f"request x has shape {tuple(req.x.shape)}, model expects {(s.seq, s.batch, s.I)}")

    def _submit(self, req: InferenceRequest, slot: int, upload_chunks: int = 0, async_outputs: bool = False) -> tuple[int, int]:
        """Enqueue one request on the current stream; returns (h2d, d2h) bytes."""
        ex = self.ex
        staging = self.staging[slot]
        host_outs = self.host_outs[slot]
        if req.x.device.type == "cpu":
            h0 = req.h0.to(torch.float32).contiguous() if req.h0 is not None else None
            c0 = req.c0.to(torch.float32).contiguous() if req.c0 is not None else None
            ex.forward_host(req.x.to(torch.float32).contiguous(), h0, c0, out_host=host_outs, staging=staging,
                            upload_chunks=upload_chunks, async_outputs=async_outputs)
            h2d = sum(t.numel() * t.element_size() for t in (req.x, h0, c0) if t is not None)
        else:
            dev = ex.device
            outs = staging[1]
            dev_t = lambda t: None if t is None else t.to(dev, torch.float32).contiguous()
            ex.forward(dev_t(req.x), dev_t(req.h0), dev_t(req.c0), out=outs)
            for dst, src in zip(host_outs, outs):
                if src is not None:
                    dst.copy_(src, non_blocking=True)
            h2d = 0
        d2h = sum(t.numel() * t.element_size() for t in staging[1] if t is not None)
        return h2d, d2h

    def run(self, req: InferenceRequest) -> InferenceResponse:
        """One request, synchronously: returns host outputs and the device
        time of H2D + forward + D2H (CUDA events)."""
        self._check(req)
        stream = torch.cuda.current_stream(self.ex.device)
        slot = self._next
        self._next = (self._next + 1) % self.slots
        self.ev[0].record(stream)
        h2d, d2h = self._submit(req, slot)
        self.ev[1].record(stream)
        self.ev[1].synchronize()
        y, hn, cn = self.host_outs[slot]
        return InferenceResponse(y, hn, cn, self.ev[0].elapsed_time(self.ev[1]), h2d, d2h)

    def run_stream(self, requests, consume=None) -> InferenceResponse:
        """Pipelined stream of requests (a serving loop).  ``consume(i, resp)``
        is called once request i's outputs are on the host, before its slot
        is reused.  Returns a summary response: the last request's outputs,
        device_ms for the whole stream, and total H2D/D2H bytes."""
        stream = torch.cuda.current_stream(self.ex.device)
        done = [None] * self.slots
        pending = [None] * self.slots
        h2d_total = d2h_total = 0

        def finish(slot):
            done[slot].synchronize()
            # host requests drain their outputs off the stream (async_outputs):
            # wait for this slot's copies, not for the requests behind it
            self.ex.outputs_ready(self.host_outs[slot][0])
            i, h2d, d2h = pending[slot]
            y, hn, cn = self.host_outs[slot]
            if consume is not None:
                consume(i, InferenceResponse(y, hn, cn, float("nan"), h2d, d2h))
            pending[slot] = None

        self.ev[0].record(stream)
        for i, req in enumerate(requests):
            self._check(req)
            slot = i % self.slots
            if pending[slot] is not None:
                finish(slot)
            # in a stream the upload overlaps the previous request: one chunk
            h2d, d2h = self._submit(req, slot, upload_chunks=1 if i else 0, async_outputs=_ASYNC_OUT)
            h2d_total += h2d
            d2h_total += d2h
            ev = done[slot] or torch.cuda.Event()
            ev.record(stream)
            done[slot] = ev
            pending[slot] = (i, h2d, d2h)
        last = None
        for k in range(self.slots):
            slot = (len(requests) + k) % self.slots
            if pending[slot] is not None:
                last = slot
                finish(slot)
        self.ev[1].record(stream)
        self.ev[1].synchronize()
        y, hn, cn = self.host_outs[last if last is not None else 0]
        return InferenceResponse(y, hn, cn, self.ev[0].elapsed_time(self.ev[1]), h2d_total, d2h_total,
                                 extra={"requests": len(requests)})


_SERVERS: dict[str, RNNServer] = {}


def register_model(name: str, executor: RNNExecutor) -> RNNServer:
    srv = RNNServer(executor)
    _SERVERS[name] = srv
    return srv


def run(request: InferenceRequest) -> InferenceResponse:
    """Run one request on the registered model ``request.model``."""
    try:
        srv = _SERVERS[request.model]
    except KeyError:
        raise ValueError(f"no model registered under {request.model!r}; call register_model first") from None
    return srv.run(request)
