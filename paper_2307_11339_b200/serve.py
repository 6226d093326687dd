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
    """Serves requests for one resident model with preallocated device input
    and pinned host output buffers (no allocation on the request path)."""

    def __init__(self, executor: RNNExecutor):
        self.ex = executor
        s = executor.spec
        dev = executor.device
        self.x_dev = torch.empty((s.seq, s.batch, s.I), device=dev)
        self.state_dev = [torch.empty((s.layers * s.dirs, s.batch, s.hidden), device=dev) for _ in range(2)]
        self.outs = executor.alloc_outputs()
        self.host_outs = [torch.empty(t.shape, dtype=t.dtype).pin_memory() if t is not None else None for t in self.outs]
        self.ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    def run(self, req: InferenceRequest) -> InferenceResponse:
        ex = self.ex
        s = ex.spec
        if tuple(req.x.shape) != (s.seq, s.batch, s.I):
            raise ValueError(f"request x has shape {tuple(req.x.shape)}, model expects {(s.seq, s.batch, s.I)}")
        stream = torch.cuda.current_stream(ex.device)
        h2d = 0
        self.ev[0].record(stream)
        self.x_dev.copy_(req.x, non_blocking=True)
        h2d += req.x.numel() * req.x.element_size() if req.x.device.type == "cpu" else 0
        states = []
        for i, st in enumerate((req.h0, req.c0)):
            if st is None:
                states.append(None)
                continue
            self.state_dev[i].copy_(st, non_blocking=True)
            h2d += st.numel() * st.element_size() if st.device.type == "cpu" else 0
            states.append(self.state_dev[i])
        ex.forward(self.x_dev, states[0], states[1], out=self.outs)
        d2h = 0
        for dst, src in zip(self.host_outs, self.outs):
            if src is not None:
                dst.copy_(src, non_blocking=True)
                d2h += src.numel() * src.element_size()
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
