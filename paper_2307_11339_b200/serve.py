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

from dataclasses import dataclass, field

import torch

from .rnn import RNNExecutor

__all__ = ["InferenceRequest", "InferenceResponse", "RNNServer", "register_model", "run"]


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
    """Serves requests for one resident model with preallocated device
    staging and pinned host output buffers (no allocation on the request
    path).  Host requests go through ``hs_rnn_forward_host``, which overlaps
    the H2D upload of x and the D2H download of y with the compute."""

    def __init__(self, executor: RNNExecutor):
        self.ex = executor
        s = executor.spec
        self.staging = executor.alloc_staging()
        self.outs = self.staging[1]
        self.host_outs = executor.alloc_host_outputs()
        self.ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    def run(self, req: InferenceRequest) -> InferenceResponse:
        ex = self.ex
        s = ex.spec
        if tuple(req.x.shape) != (s.seq, s.batch, s.I):
            raise ValueError(f"request x has shape {tuple(req.x.shape)}, model expects {(s.seq, s.batch, s.I)}")
        stream = torch.cuda.current_stream(ex.device)
        on_host = req.x.device.type == "cpu"
        h2d = 0
        self.ev[0].record(stream)
        if on_host:
            h0 = req.h0.contiguous() if req.h0 is not None else None
            c0 = req.c0.contiguous() if req.c0 is not None else None
            ex.forward_host(req.x.contiguous(), h0, c0, out_host=self.host_outs, staging=self.staging)
            h2d = sum(t.numel() * t.element_size() for t in (req.x, h0, c0) if t is not None)
        else:
            dev = ex.device
            ex.forward(req.x, None if req.h0 is None else req.h0.to(dev), None if req.c0 is None else req.c0.to(dev),
                       out=self.outs)
            for dst, src in zip(self.host_outs, self.outs):
                if src is not None:
                    dst.copy_(src, non_blocking=True)
        d2h = sum(t.numel() * t.element_size() for t in self.outs if t is not None)
        self.ev[1].record(stream)
        self.ev[1].synchronize()
        y, hn, cn = self.host_outs
        return InferenceResponse(y, hn, cn, self.ev[0].elapsed_time(self.ev[1]), h2d, d2h)


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
