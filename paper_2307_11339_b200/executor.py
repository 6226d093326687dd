"""Real execution of a partition plan and the measured per-operator profile.

These are the two seams of the reference that change:

* :func:`execute` replaces the virtual-time replay ``engine.simulate``
  (/root/reference/pkg/src/hetsched/engine.py:265-418).  It consumes the same
  ``(Graph, Plan)`` pair and returns real tensors plus a :class:`Trace` whose
  spans are measured (CUDA events for GPU work, ``perf_counter`` for host
  cores).  Semantics kept from the reference: each processor drains its
  nodes in plan order (engine.py:287-289), a node starts once all its inputs
  have arrived (engine.py:359-372), and crossing edges move data over the
  PCIe link (engine.py:320-328) — here as real pinned-memory copies.
* :func:`profile_ops` replaces the seeded generator ``synth_profile``
  (costmodel.py:176-221): it fills the same ``W``/``C``/``Mem``/``b`` tables
  from B200 CUDA-event timings, host-core timings under ``j``-way contention
  and the real tensor sizes.

Execution modes of :func:`execute`:

* all-GPU plan (``k_star == 0``, the reference's "GPU" pattern and the
  latency-optimal plan whenever the B200 dominates): ONE fused forward through
  ``hs_rnn_forward_packed`` — K1 tensor-core input GEMMs plus the persistent
  recurrent wavefront.  Per-node spans apportion each layer's measured time
  evenly over its cells.
* hybrid plan (Chrion's CPU/GPU co-execution): maximal runs
  of consecutive GPU cells of one layer-direction become ``hs_rnn_run_cells``
  segments on the GPU stream; host cells run on ``k_star`` worker threads (one
  per plan core, PyTorch fp32 CPU ops, one intra-op thread each); crossing
  edges are pinned-memory copies on a dedicated copy stream.  Host cells exist
  only because the plan puts them there — the GPU side has no CPU fallback.
"""
from __future__ import annotations

import os
import statistics
import sys
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from .costmodel import CostModel, snap_mem
from .engine import GPU, NodeSpan, Trace, TransferSpan
from .graph import Graph, gen_bilstm_grid, gen_lstm_grid, grid_cell

__all__ = [
    "HostRNN",
    "ExecResult",
    "Schedule",
    "GpuSegment",
    "build_schedule",
    "check_grid",
    "execute",
    "profile_ops",
    "measure_link_bandwidth",
    "measure_link_latency",
]

MB = float(2**20)


# --------------------------------------------------------------- host cells
class HostRNN:
    """Host-core cell evaluator for the CPU side of hybrid plans.

    Weights are kept transposed and contiguous in fp32 so a cell is two
    ``addmm`` calls plus the gate update (PyTorch LSTM i,f,g,o / GRU r,z,n).
    """

    def __init__(self, spec, weights):
        self.spec = spec
        self.w = []
        for w in weights:
            self.w.append({
                "w_ihT": w["w_ih"].detach().to("cpu", torch.float32).t().contiguous(),
                "w_hhT": w["w_hh"].detach().to("cpu", torch.float32).t().contiguous(),
                "b_ih": w["b_ih"].detach().to("cpu", torch.float32).contiguous(),
                "b_hh": w["b_hh"].detach().to("cpu", torch.float32).contiguous(),
            })

    def cell(self, ld: int, xin: torch.Tensor, hp: torch.Tensor, cp: torch.Tensor | None):
        """One cell of layer-direction ``ld``: returns (h_t, c_t) (c_t None for GRU)."""
        w = self.w[ld]
        H = self.spec.hidden
        gx = torch.addmm(w["b_ih"], xin, w["w_ihT"])
        gh = torch.addmm(w["b_hh"], hp, w["w_hhT"])
        if self.spec.cell == "lstm":
            g = gx.add_(gh)
            i = torch.sigmoid(g[:, :H])
            f = torch.sigmoid(g[:, H:2 * H])
            gg = torch.tanh(g[:, 2 * H:3 * H])
            o = torch.sigmoid(g[:, 3 * H:])
            c = f * cp + i * gg
            return o * torch.tanh(c), c
        r = torch.sigmoid(gx[:, :H] + gh[:, :H])
        z = torch.sigmoid(gx[:, H:2 * H] + gh[:, H:2 * H])
        n = torch.tanh(gx[:, 2 * H:] + r * gh[:, 2 * H:])
        return (1.0 - z) * n + z * hp, None


def _host_model(model):
    from .rnn import RNNExecutor

    if isinstance(model, HostRNN):
        return model
    if isinstance(model, RNNExecutor):
        if getattr(model, "_host", None) is None:
            model._host = HostRNN(model.spec, model.weights)
        return model._host
    raise TypeError("model must be an RNNExecutor or a HostRNN")


# ------------------------------------------------------------- graph checks
_GRID_CACHE: dict = {}


def check_grid(graph: Graph, spec) -> None:
    """Raise ValueError unless ``graph`` is exactly the unrolled cell grid of
    ``spec`` (``gen_lstm_grid`` / ``gen_bilstm_grid`` numbering)."""
    L, T, D = spec.layers, spec.seq, spec.dirs
    if graph.n != L * D * T:
        raise ValueError(f"graph has {graph.n} nodes; the {L}x{D}x{T} cell grid has {L * D * T}")
    key = (L, T, D)
    want = _GRID_CACHE.get(key)
    if want is None:
        want = (gen_lstm_grid(L, T) if D == 1 else gen_bilstm_grid(L, T)).edge_set
        _GRID_CACHE[key] = want
    if graph.edge_set != want:
        raise ValueError("graph is not the layers x timesteps cell grid of this RNN")


def _check_plan(graph: Graph, plan) -> None:
    n = graph.n
    seq = plan.order.seq
    if len(seq) != n or sorted(seq) != list(range(n)):
        raise ValueError("plan order is not a permutation of the graph's nodes")
    if len(plan.selection) != n or len(plan.cores) != n:
        raise ValueError("plan selection/cores do not match the graph size")
    pos = [0] * n
    for i, v in enumerate(seq):
        pos[v] = i
    for s, d in graph.edge_set:
        if pos[s] > pos[d]:
            raise ValueError(f"plan order visits node {d} before its predecessor {s}")
    for v in range(n):
        if plan.selection[v] not in (0, 1):
            raise ValueError(f"selection[{v}] must be 0 (GPU) or 1 (host)")
        if plan.selection[v] == 1 and not 1 <= plan.cores[v] <= max(plan.k_star, 0):
            raise ValueError(f"host node {v} is pinned to core {plan.cores[v]} outside 1..k_star={plan.k_star}")


# ----------------------------------------------------------------- schedule
@dataclass(frozen=True)
class GpuSegment:
    """Processing steps ``s0..s1-1`` of layer-direction ``ld`` on the GPU."""

    ld: int
    s0: int
    s1: int
    nodes: tuple[int, ...]


@dataclass(frozen=True)
class Schedule:
    gpu: tuple[GpuSegment, ...]
    host: dict            # core -> tuple of nodes in plan order
    cells: tuple          # node -> (l, d, t, s)
    host_consumed: frozenset  # GPU nodes whose output a host node reads
    gpu_consumed: frozenset   # host nodes whose output a GPU node reads


def build_schedule(graph: Graph, plan, spec) -> Schedule:
    """Split a plan into GPU segments and per-core host queues.

    A GPU node joins the open segment only if it is the next processing step
    of the same layer-direction, directly follows it in the GPU queue, and has
    no host predecessor.  Only a segment's first node can then wait on host
    cells, and those precede it in the (topological) plan order, so every
    processor draining its queue in plan order cannot deadlock.
    """
    check_grid(graph, spec)
    _check_plan(graph, plan)
    T, D = spec.seq, spec.dirs
    cells = []
    for v in range(graph.n):
        l, d, t = grid_cell(v, T, D)
        cells.append((l, d, t, t if d == 0 else T - 1 - t))
    sel = plan.selection
    pred = graph.pred
    segs: list[list] = []
    host: dict[int, list[int]] = {}
    for v in plan.order.seq:
        l, d, t, s = cells[v]
        if sel[v] == GPU:
            ld = l * D + d
            host_pred = any(sel[m] != GPU for m in pred[v])
            if segs and not host_pred:
                cur = segs[-1]
                if cur[0] == ld and cur[2] == s:
                    cur[2] = s + 1
                    cur[3].append(v)
                    continue
            segs.append([ld, s, s + 1, [v]])
        else:
            host.setdefault(plan.cores[v], []).append(v)
    host_consumed = set()
    gpu_consumed = set()
    for a, b in graph.edge_set:
        if (sel[a] == GPU) != (sel[b] == GPU):
            (host_consumed if sel[a] == GPU else gpu_consumed).add(a)
    return Schedule(
        gpu=tuple(GpuSegment(ld, s0, s1, tuple(ns)) for ld, s0, s1, ns in segs),
        host={c: tuple(q) for c, q in host.items()},
        cells=tuple(cells),
        host_consumed=frozenset(host_consumed),
        gpu_consumed=frozenset(gpu_consumed),
    )


@dataclass
class ExecResult:
    """Outputs of one plan execution.  ``trace.makespan`` follows the
    reference's definition (engine.py:408-415): the last node's end, or a
    host-bound transfer's; ``wall_ms`` is the whole call as the caller sees
    it, including the final assembly of host-produced rows into ``y`` /
    ``h_n`` / ``c_n`` on the device."""

    y: torch.Tensor
    hn: torch.Tensor
    cn: torch.Tensor | None
    trace: Trace
    wall_ms: float = 0.0


# ------------------------------------------------------------------ execute
def execute(graph: Graph, plan, model, x: torch.Tensor, h0=None, c0=None) -> ExecResult:
    """Run ``plan`` over the RNN's cell grid with real tensors.

    ``model`` is an :class:`~paper_2307_11339_b200.rnn.RNNExecutor` (needed
    whenever the plan places a node on the GPU) or a :class:`HostRNN` (all-host
    plans).  ``x`` is ``[T, B, I]``; ``h0``/``c0`` ``[L*D, B, H]`` or None.
    Returns ``(y, h_n, c_n, trace)``; tensors live on the GPU when the plan
    uses it, else on the host.
    """
    from .rnn import RNNExecutor

    spec = model.spec
    sched = build_schedule(graph, plan, spec)
    uses_gpu = bool(sched.gpu)
    if uses_gpu and not isinstance(model, RNNExecutor):
        raise ValueError("plan places nodes on the GPU: pass an RNNExecutor")
    if tuple(x.shape) != (spec.seq, spec.batch, spec.I):
        raise ValueError(f"x has shape {tuple(x.shape)}, expected {(spec.seq, spec.batch, spec.I)}")
    if uses_gpu and not sched.host:
        return _execute_fused(graph, sched, model, x, h0, c0)
    return _execute_hybrid(graph, plan, sched, model, x, h0, c0)


def _execute_fused(graph, sched, ex, x, h0, c0) -> ExecResult:
    spec = ex.spec
    dev = ex.device
    x = x.to(dev, torch.float32).contiguous()
    h0 = h0.to(dev, torch.float32).contiguous() if h0 is not None else None
    c0 = c0.to(dev, torch.float32).contiguous() if c0 is not None else None
    t0 = time.perf_counter()
    y, hn, cn, lm = ex.forward(x, h0, c0, layer_ms=True)
    torch.cuda.synchronize(dev)
    wall = (time.perf_counter() - t0) * 1e3
    T, D = spec.seq, spec.dirs
    spans = []
    off = 0.0
    for l, (g_ms, r_ms) in enumerate(lm):
        dt = (g_ms + r_ms) / T
        for d in range(D):
            for t in range(T):
                s = t if d == 0 else T - 1 - t
                v = (l * D + d) * T + t
                spans.append(NodeSpan(v, GPU, off + s * dt, off + (s + 1) * dt))
        off += g_ms + r_ms
    spans.sort(key=lambda sp: (sp.start, sp.node))
    return ExecResult(y, hn, cn, Trace(nodes=tuple(spans), transfers=(), makespan=off), wall_ms=wall)


class _Failure:
    def __init__(self):
        self.exc = None
        self.lock = threading.Lock()

    def set(self, exc):
        with self.lock:
            if self.exc is None:
                self.exc = exc


def _wait(evt: threading.Event, fail: _Failure):
    while not evt.wait(0.05):
        if fail.exc is not None:
            raise RuntimeError("hybrid execution aborted") from fail.exc


_POOL = None
_POOL_LOCK = threading.Lock()


def _worker_pool(n: int):
    """Process-wide pool of plan workers (one thread per host core of a plan,
    plus the GPU queue's).  Threads persist across ``execute`` calls: a fresh
    thread per call cost ~0.3 ms to start and ~0.4 ms more for its first
    cell (per-thread runtime setup), which the cost model has no term for."""
    global _POOL
    from concurrent.futures import ThreadPoolExecutor

    with _POOL_LOCK:
        if _POOL is None or _POOL._max_workers < n:
            old = _POOL
            _POOL = ThreadPoolExecutor(max_workers=max(n, 4), thread_name_prefix="hs-plan",
                                       initializer=torch.set_num_threads, initargs=(1,))
            if old is not None:
                old.shutdown(wait=False)
        return _POOL


def _execute_hybrid(graph, plan, sched: Schedule, model, x, h0, c0) -> ExecResult:
    spec = model.spec
    host_rnn = _host_model(model)
    L, D, T, B, H = spec.layers, spec.dirs, spec.seq, spec.batch, spec.hidden
    LD = L * D
    lstm = spec.cell == "lstm"
    uses_gpu = bool(sched.gpu)
    pin = uses_gpu

    def hbuf(*shape):
        t = torch.zeros(shape, dtype=torch.float32)
        return t.pin_memory() if pin else t

    # host mirrors (write-once per cell slot)
    x_host = x.detach().to("cpu", torch.float32).contiguous()
    if pin:
        x_host = x_host.pin_memory()
    act_h = [hbuf(T, B, D * H) for _ in range(L)]
    hs_h = [hbuf(T, B, H) for _ in range(LD)]
    cs_h = [hbuf(T, B, H) for _ in range(LD)] if lstm else None
    h0_h = h0.detach().to("cpu", torch.float32) if h0 is not None else torch.zeros(LD, B, H)
    c0_h = (c0.detach().to("cpu", torch.float32) if c0 is not None else torch.zeros(LD, B, H)) if lstm else None

    n = graph.n
    cells = sched.cells
    sel = plan.selection
    pred = graph.pred
    succ = graph.succ
    ready = [threading.Event() for _ in range(n)]       # host-visible output
    d2h_evt: list = [None] * n
    fail = _Failure()
    t_start = time.perf_counter()
    host_spans: list[NodeSpan] = []
    spans_lock = threading.Lock()

    # ------------------------------------------------------------ GPU side
    if uses_gpu:
        ex = model
        dev = ex.device
        stream = torch.cuda.Stream(dev)
        copy_stream = torch.cuda.Stream(dev)
        with torch.cuda.device(dev):
            x_dev = x_host.to(dev, non_blocking=True)
            act_d = [torch.zeros((T, B, D * H), device=dev) for _ in range(L)]
            hs_d = [torch.zeros((T, B, H), device=dev) for _ in range(LD)]
            cs_d = [torch.zeros((T, B, H), device=dev) for _ in range(LD)] if lstm else None
            h0_d = h0_h.to(dev)
            c0_d = c0_h.to(dev) if lstm else None
            ev0 = torch.cuda.Event(enable_timing=True)
            # every timing event of the run, created (and its CUDA event
            # materialised) before the clock starts: per segment 2, per
            # crossing 2
            n_ev = 2 * len(sched.gpu) + 2 * sum(1 for seg in sched.gpu for v in seg.nodes if v in sched.host_consumed) + \
                2 * sum(1 for seg in sched.gpu for m in pred[seg.nodes[0]] if sel[m] != GPU)
            ev_pool = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
            for e in ev_pool + [ev0]:
                e.record(stream)
            torch.cuda.synchronize(dev)
            ev_pool.reverse()
        seg_events = []
        xfer_events = []  # (src, dst, start_evt, end_evt, mb)

    def state_slice(ld, s, side):
        """(h, c) of layer-direction ld after processing step s on `side`."""
        if s < 0:
            src = (h0_d, c0_d) if side == "d" else (h0_h, c0_h)
            return src[0][ld], (src[1][ld] if lstm else None)
        if side == "d":
            return hs_d[ld][s], (cs_d[ld][s] if lstm else None)
        return hs_h[ld][s], (cs_h[ld][s] if lstm else None)

    def take_ev():  # a pre-made timing event (a fresh one if the count was short)
        return ev_pool.pop() if ev_pool else torch.cuda.Event(enable_timing=True)

    def gpu_worker():  # runs on the calling thread, inside the device / stream context
        try:
            for seg in sched.gpu:
                ld, s0, s1 = seg.ld, seg.s0, seg.s1
                l, d = divmod(ld, D)
                first = seg.nodes[0]
                # host-produced inputs of the first node: wait, then H2D
                for m in pred[first]:
                    if sel[m] == GPU:
                        continue
                    _wait(ready[m], fail)
                    ml, md, mt, ms = cells[m]
                    e0, e1 = take_ev(), take_ev()
                    e0.record(stream)
                    if ml == l and md == d:  # state edge
                        hs_d[ld][ms].copy_(hs_h[ld][ms], non_blocking=True)
                        nbytes = B * H * 4
                        if lstm:
                            cs_d[ld][ms].copy_(cs_h[ld][ms], non_blocking=True)
                            nbytes *= 2
                    else:  # layer-input edge
                        sl = slice(md * H, (md + 1) * H)
                        act_d[ml][mt, :, sl].copy_(act_h[ml][mt, :, sl], non_blocking=True)
                        nbytes = B * H * 4
                    e1.record(stream)
                    xfer_events.append((m, first, e0, e1, nbytes / MB))
                inp = x_dev if l == 0 else act_d[l - 1]
                h_prev, c_prev = state_slice(ld, s0 - 1, "d")
                h_last, c_last = state_slice(ld, s1 - 1, "d")
                e0, e1 = take_ev(), take_ev()
                e0.record(stream)
                ex.run_cells(ld, s0, s1, inp, act_d[l], h_prev, c_prev if lstm else None, h_last, c_last,
                             stream=stream)
                e1.record(stream)
                seg_events.append((seg, e0, e1))
                # outputs that host cells read: D2H on the copy stream
                for v in seg.nodes:
                    if v not in sched.host_consumed:
                        continue
                    vl, vd, vt, vs = cells[v]
                    copy_stream.wait_event(e1)
                    c0e, c1e = take_ev(), take_ev()
                    c0e.record(copy_stream)
                    with torch.cuda.stream(copy_stream):
                        nbytes = 0
                        for w in succ[v]:
                            if sel[w] == GPU:
                                continue
                            wl, wd, _wt, _ws = cells[w]
                            if wl == vl and wd == vd:
                                if vs != s1 - 1:
                                    raise AssertionError("state edge leaves a GPU segment mid-way")
                                hs_h[ld][vs].copy_(hs_d[ld][vs], non_blocking=True)
                                nbytes += B * H * 4
                                if lstm:
                                    cs_h[ld][vs].copy_(cs_d[ld][vs], non_blocking=True)
                                    nbytes += B * H * 4
                            else:
                                sl = slice(vd * H, (vd + 1) * H)
                                act_h[vl][vt, :, sl].copy_(act_d[vl][vt, :, sl], non_blocking=True)
                                nbytes += B * H * 4
                    c1e.record(copy_stream)
                    d2h_evt[v] = c1e
                    xfer_events.append((v, -1, c0e, c1e, nbytes / MB))
                    ready[v].set()
        except BaseException as exc:  # surface in the caller
            fail.set(exc)

    # ----------------------------------------------------------- host side
    def host_worker(core, queue):
        try:
            for v in queue:
                l, d, t, s = cells[v]
                ld = l * D + d
                for m in pred[v]:
                    _wait(ready[m], fail)
                    if sel[m] == GPU:
                        d2h_evt[m].synchronize()
                t0 = time.perf_counter()
                xin = x_host[t] if l == 0 else act_h[l - 1][t]
                hp, cp = state_slice(ld, s - 1, "h")
                h, c = host_rnn.cell(ld, xin, hp, cp)
                act_h[l][t, :, d * H:(d + 1) * H] = h
                hs_h[ld][s] = h
                if lstm:
                    cs_h[ld][s] = c
                t1 = time.perf_counter()
                with spans_lock:
                    host_spans.append(NodeSpan(v, core, (t0 - t_start) * 1e3, (t1 - t_start) * 1e3))
                ready[v].set()
        except BaseException as exc:
            fail.set(exc)

    # cells hand off between worker threads at every crossing: a short GIL
    # switch interval (default 5 ms) keeps a woken waiter from queueing behind
    # a running worker for a whole interval
    prev_switch = sys.getswitchinterval()
    sys.setswitchinterval(5e-5)
    tasks = [(host_worker, (c, q)) for c, q in sorted(sched.host.items())]
    pool = _worker_pool(len(tasks))
    if uses_gpu:
        # the GPU queue runs on the calling thread (no hand-off before its
        # first launch), inside its device / stream context entered before
        # the clock starts
        with torch.cuda.device(dev), torch.cuda.stream(stream):
            t_start = time.perf_counter()
            ev0.record(stream)
            futs = [pool.submit(fn, *args) for fn, args in tasks]
            gpu_worker()
    else:
        t_start = time.perf_counter()
        futs = [pool.submit(fn, *args) for fn, args in tasks]
    for fut in futs:
        fut.result()
    sys.setswitchinterval(prev_switch)
    if fail.exc is not None:
        raise RuntimeError("hybrid plan execution failed") from fail.exc

    # ---------------------------------------------------------- assemble
    spans = list(host_spans)
    transfers = []
    if uses_gpu:
        with torch.cuda.device(dev):
            # host-produced final outputs -> device y / h_n / c_n
            torch.cuda.synchronize(dev)
            y = act_d[L - 1]
            # host-produced rows of the output: one upload of the host mirror and
            # one masked select instead of a copy per cell
            mask = torch.zeros((T, 1, D * H), dtype=torch.bool)
            for v in range(n):
                l, d, t, s = cells[v]
                if sel[v] != GPU and l == L - 1:
                    mask[t, 0, d * H:(d + 1) * H] = True
            if bool(mask.any()):
                y = torch.where(mask.to(dev, non_blocking=True), act_h[L - 1].to(dev, non_blocking=True), y)
            hn = torch.empty((LD, B, H), device=dev)
            cn = torch.empty((LD, B, H), device=dev) if lstm else None
            for ld in range(LD):
                l, d = divmod(ld, D)
                t_last = T - 1 if d == 0 else 0
                v = ld * T + t_last
                side = "d" if sel[v] == GPU else "h"
                h, c = state_slice(ld, T - 1, side)
                hn[ld].copy_(h)
                if lstm:
                    cn[ld].copy_(c)
            torch.cuda.synchronize(dev)
        end_ms = (time.perf_counter() - t_start) * 1e3
        for seg, e0, e1 in seg_events:
            a, b = ev0.elapsed_time(e0), ev0.elapsed_time(e1)
            k = len(seg.nodes)
            for i, v in enumerate(seg.nodes):
                spans.append(NodeSpan(v, GPU, a + (b - a) * i / k, a + (b - a) * (i + 1) / k))
        for src, dst, e0, e1, mb in xfer_events:
            transfers.append(TransferSpan(src, dst, ev0.elapsed_time(e0), ev0.elapsed_time(e1), mb))
    else:
        end_ms = (time.perf_counter() - t_start) * 1e3
        y = act_h[L - 1]
        hn = torch.stack([state_slice(ld, T - 1, "h")[0] for ld in range(LD)]).clone()
        cn = torch.stack([state_slice(ld, T - 1, "h")[1] for ld in range(LD)]).clone() if lstm else None
    # the reference's makespan (engine.py:408-415): last node end, or the end
    # of a host-bound output transfer; the assembly above is in wall_ms only
    makespan = max([sp.end for sp in spans] + [tr.end for tr in transfers if tr.dst < 0])
    spans.sort(key=lambda sp: (sp.start, sp.node))
    transfers.sort(key=lambda x: (x.start, x.src, x.dst))
    return ExecResult(y, hn, cn, Trace(nodes=tuple(spans), transfers=tuple(transfers), makespan=makespan),
                      wall_ms=max(end_ms, makespan))


# ----------------------------------------------------------------- profiler
def measure_link_bandwidth(device, nbytes: int = 64 * 2**20, reps: int = 5) -> float:
    """Pinned host->device copy bandwidth in MB/ms (the cost model's ``b``)."""
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=device)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return (nbytes / MB) / statistics.median(ts)


def measure_link_latency(device, reps: int = 20) -> float:
    """Fixed cost (ms) of one plan-boundary crossing as ``execute`` performs it:
    a small pinned device->host copy on a copy stream and the host thread's
    wait on its event (the reference's comm_time has only the byte term,
    costmodel.py:133-139; profile_ops folds this latency into C so the
    planner's crossing cost is the measured one)."""
    src = torch.zeros(256, device=device)
    dst = torch.empty(256).pin_memory()
    st = torch.cuda.Stream(device)
    ts = []
    for _ in range(reps + 2):
        ev = torch.cuda.Event()
        t0 = time.perf_counter()
        with torch.cuda.stream(st):
            dst.copy_(src, non_blocking=True)
            ev.record(st)
        ev.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts[2:])


def _host_cell_ms(host_rnn: HostRNN, ld: int, j: int, reps: int) -> float:
    """Median ms of one host cell of layer-direction ``ld`` while ``j`` cells
    run concurrently on ``j`` single-threaded workers (the reference's
    "time when j cores are busy" column, costmodel.py:47-61).  Timed as the
    hybrid executor's host worker runs a cell: the cell's ops plus the writes
    of its outputs into the host activation and state mirrors."""
    spec = host_rnn.spec
    l = ld // spec.dirs
    d = ld % spec.dirs
    H = spec.hidden
    gen = torch.Generator().manual_seed(ld)
    xin = torch.rand((spec.batch, spec.layer_input(l)), generator=gen)
    hp = torch.rand((spec.batch, H), generator=gen)
    cp = hp.clone() if spec.cell == "lstm" else None
    times = [[] for _ in range(j)]
    barrier = threading.Barrier(j)

    def work(i):
        torch.set_num_threads(1)
        act = torch.zeros((2, spec.batch, spec.dirs * H))
        hs_ = torch.zeros((2, spec.batch, H))
        cs_ = torch.zeros((2, spec.batch, H))
        host_rnn.cell(ld, xin, hp, cp)
        for _ in range(reps):
            barrier.wait()
            t0 = time.perf_counter()
            h, c = host_rnn.cell(ld, xin, hp, cp)
            act[1, :, d * H:(d + 1) * H] = h
            hs_[1] = h
            if c is not None:
                cs_[1] = c
            times[i].append((time.perf_counter() - t0) * 1e3)

    prev = torch.get_num_threads()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(j)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    torch.set_num_threads(prev)
    return statistics.median(x for ts in times for x in ts)


def profile_ops(graph: Graph, model, k: int | None = None, reps: int = 5, b: float | None = None) -> CostModel:
    """Measured cost model of the RNN cell grid (drop-in for ``synth_profile``).

    * ``W[:, 0]``: B200 ms per cell from ``hs_rnn_profile_cells`` — each
      cell's measured recurrence step (per-step %globaltimer stamps), scaled
      so the cells sum to the measured forward (CUDA events), median of
      ``reps``.  An all-GPU plan's modelled latency therefore equals the
      measured forward, and the split between cells follows
      the measured steps (e.g. the wavefront's pipeline fill).  Hybrid plans'
      GPU segments run the fused forward's own kernels (``hs_rnn_run_cells``: tensor-core, or the small-shape cluster kernel).
      Needs an RNNExecutor; with a HostRNN the GPU column is the host column
      x 1e3 so no plan selects the GPU.
    * ``W[:, j]``, j = 1..k: host ms per cell with ``j`` cells running at once.
    * ``C[m, i]``: MB moved on each edge (h, plus c on LSTM state edges),
      plus the measured per-crossing latency x ``b`` (``measure_link_latency``),
      so ``comm_time = C / b`` (costmodel.py:133-139) is bytes / b + latency.
    * ``Mem[i]``: (input, output, ephemeral gates, weights) MB, on MEM_GRID.
    * ``b``: measured pinned H2D MB/ms (or the given value).
    """
    from .rnn import RNNExecutor

    spec = model.spec
    check_grid(graph, spec)
    host_rnn = _host_model(model)
    L, D, T, B, H, G = spec.layers, spec.dirs, spec.seq, spec.batch, spec.hidden, spec.G
    n = graph.n
    if k is None:
        k = max(1, min(4, (os.cpu_count() or 2) - 1))
    lstm = spec.cell == "lstm"
    # host columns: one measurement per distinct input width (layer 0 vs l>=1)
    host_ms = {}
    for ld in range(L * D):
        key = spec.layer_input(ld // D)
        if key not in host_ms:
            host_ms[key] = [_host_cell_ms(host_rnn, ld, j, reps) for j in range(1, k + 1)]
    W = np.empty((n, k + 1))
    for v in range(n):
        l = (v // T) // D
        W[v, 1:] = host_ms[spec.layer_input(l)]
    if isinstance(model, RNNExecutor):
        dev = model.device
        x = torch.rand((T, B, spec.I), generator=torch.Generator().manual_seed(1)).to(dev)
        outs = model.alloc_outputs()
        model.forward(x, out=outs)
        runs = [model.profile_cells(x, out=outs)[0] for _ in range(reps)]
        W[:, 0] = np.median(np.asarray(runs, dtype=np.float64), axis=0)
        if b is None:
            b = measure_link_bandwidth(dev)
        lat_ms = measure_link_latency(dev)
    else:
        W[:, 0] = W[:, 1] * 1e3
        if b is None:
            b = 16.0
        lat_ms = 0.0
    C = np.zeros((n, n))
    for s, d in graph.edge_set:
        same_chain = (s // T) == (d // T)
        C[s, d] = (B * H * 4 * (2 if (lstm and same_chain) else 1)) / MB + lat_ms * b
    Mem = np.empty((n, 4))
    for v in range(n):
        l = (v // T) // D
        Il = spec.layer_input(l)
        Mem[v] = [
            B * Il * 4 / MB,
            B * H * 4 * (2 if lstm else 1) / MB,
            B * G * H * 4 / MB,
            (G * H * (Il + H) + 2 * G * H) * 4 / MB,
        ]
    return CostModel(k=k, b=float(b), W=W, C=C, Mem=snap_mem(Mem), c_edges=frozenset(graph.edge_set))
