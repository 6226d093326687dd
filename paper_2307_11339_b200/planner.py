"""Partition planning (drop-in for ``hetsched.planner``).

Algorithm 1 (:func:`topo_sort_hybrid`): FIFO ready queue with transfer-aware
depth-first chaining.  Algorithm 2 (:func:`sweep_core_counts` /
:func:`select_devices`): for every host core budget k' in 0..k, place each node
(in plan order) on the processor minimising ``EFT + alpha * dM`` and keep the
budget with the lowest ``latency + alpha * memory``.  Plans are bit-exact with
the reference: identical float expressions in identical order, strict ``<``
ties preferring the GPU, then the lowest core, then the lowest budget
(SURVEY §7.3 H8).

New here: :func:`sweep_alpha` (the latency/memory
frontier of ``hetsched sweep``) and :func:`memory_optimal_alpha` (the largest
alpha whose latency still meets the SLO — the reference has no chooser).

Reference anchors: Order/Plan planner.py:46-63, topo_sort_bfs 73-88,
topo_sort_dfs 91-119, topo_sort_hybrid 122-185, sweep_core_counts 199-275,
select_devices 278-292, crossing_count 295-300, reduce_movements 303-356,
check_plan 359-365, plan JSON 368-408; sweep CLI cli.py:259-306.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, replace
from pathlib import Path
from typing import TYPE_CHECKING

from . import engine
from .costmodel import CostModel, check_compatible

if TYPE_CHECKING:
    from .graph import Graph

__all__ = [
    "Order",
    "Plan",
    "PlanFormatError",
    "CoreCountPoint",
    "AlphaPoint",
    "topo_sort_bfs",
    "topo_sort_dfs",
    "topo_sort_hybrid",
    "select_devices",
    "sweep_core_counts",
    "sweep_alpha",
    "memory_optimal_alpha",
    "latency_optimal_plan",
    "reduce_movements",
    "check_plan",
    "crossing_count",
    "save_plan",
    "load_plan",
]


class PlanFormatError(ValueError):
    """A plan file is unparsable or inconsistent."""


@dataclass(frozen=True)
class Order:
    seq: tuple[int, ...]


@dataclass(frozen=True)
class Plan:
    """Visit order, device class per node (0 GPU / 1 host), processor per node,
    host core budget and the memory weight alpha the plan was built for."""

    order: Order
    selection: tuple[int, ...]
    cores: tuple[int, ...]
    k_star: int
    alpha: float


def _require_complete(graph: "Graph", produced: int) -> None:
    if produced != graph.n:
        raise ValueError("graph contains a cycle; topological ordering is impossible")


def topo_sort_bfs(graph: "Graph") -> Order:
    """Kahn's algorithm with a FIFO queue seeded in ascending index order."""
    missing = [len(p) for p in graph.pred]
    fifo = [v for v in range(graph.n) if missing[v] == 0]
    head = 0
    while head < len(fifo):
        u = fifo[head]
        head += 1
        for v in graph.succ[u]:
            missing[v] -= 1
            if missing[v] == 0:
                fifo.append(v)
    _require_complete(graph, len(fifo))
    return Order(seq=tuple(fifo))


def topo_sort_dfs(graph: "Graph") -> Order:
    """Depth-first from each entry (ascending); a child is entered only once
    all of its predecessors have been emitted."""
    placed = [False] * graph.n
    seq: list[int] = []
    pred, succ = graph.pred, graph.succ
    for root in range(graph.n):
        if placed[root] or pred[root]:
            continue
        placed[root] = True
        seq.append(root)
        frames = [[root, 0]]
        while frames:
            top = frames[-1]
            kids = succ[top[0]]
            if top[1] >= len(kids):
                frames.pop()
                continue
            c = kids[top[1]]
            top[1] += 1
            if not placed[c] and all(placed[m] for m in pred[c]):
                placed[c] = True
                seq.append(c)
                frames.append([c, 0])
    _require_complete(graph, len(seq))
    return Order(seq=tuple(seq))


def topo_sort_hybrid(graph: "Graph", cm: CostModel) -> Order:
    """Algorithm 1: ready-queue order with transfer-aware chaining.

    A node popped from the FIFO is emitted once all its predecessors are
    emitted (else it is re-queued at the tail).  After emitting u, its
    children are scanned depth-first: a child with a single predecessor whose
    boundary transfer ``C[u,c]/b`` strictly exceeds the mean of its GPU time
    and its full-budget host time is emitted immediately; any other child
    not yet queued joins the FIFO.
    """
    check_compatible(graph, cm)
    n, k = graph.n, cm.k
    b = float(cm.b)
    W = cm.W
    C = cm.C
    pred, succ = graph.pred, graph.succ
    emitted = [False] * n
    queued = [False] * n
    seq: list[int] = []
    fifo: list[int] = []

    def worth_chaining(u: int, c: int) -> bool:
        mean_exec = (float(W[c, 0]) + float(W[c, k])) / 2.0
        return len(pred[c]) == 1 and float(C[u, c]) / b > mean_exec

    def emit_with_chain(v: int) -> None:
        emitted[v] = True
        seq.append(v)
        frames = [[v, 0]]
        while frames:
            top = frames[-1]
            kids = succ[top[0]]
            if top[1] >= len(kids):
                frames.pop()
                continue
            c = kids[top[1]]
            top[1] += 1
            if emitted[c]:
                continue
            if worth_chaining(top[0], c):
                emitted[c] = True
                seq.append(c)
                frames.append([c, 0])
            elif not queued[c]:
                queued[c] = True
                fifo.append(c)

    for v in graph.entries:
        queued[v] = True
        fifo.append(v)
    head = 0
    blocked_run = 0
    while head < len(fifo):
        u = fifo[head]
        head += 1
        if emitted[u]:
            continue
        if all(emitted[m] for m in pred[u]):
            emit_with_chain(u)
            blocked_run = 0
            continue
        fifo.append(u)
        blocked_run += 1
        if blocked_run > len(fifo) - head:
            break  # everything still queued is blocked: a cycle
    _require_complete(graph, len(seq))
    return Order(seq=tuple(seq))


@dataclass(frozen=True)
class CoreCountPoint:
    k_prime: int
    plan: Plan
    latency: float
    gpu_memory: float
    total_cost: float


def _greedy_for_budget(graph, cm, order, alpha, k_prime, io_transfers, tables):
    """One pass of Algorithm 2 at host budget ``k_prime``."""
    W, mem, inc, b, entries = tables
    pred = graph.pred
    n = graph.n
    free = [0.0] * (k_prime + 1)
    aft = [0.0] * n
    classes = [0] * n
    cores = [0] * n
    for v in order.seq:
        row = mem[v]
        dmem = row[1] + row[2] + row[3]
        for m in pred[v]:
            if classes[m] != engine.GPU:
                dmem += mem[m][1]
        is_entry = v in entries
        ccol = inc[v]
        best_j, best_cost, best_f = -1, 0.0, 0.0
        for j in range(k_prime + 1):
            cls = 0 if j == 0 else 1
            w = W[v][0] if j == 0 else W[v][k_prime]
            rdy = engine._input_ready(row, b, cls, is_entry, io_transfers)
            _s, f = engine.step_times(pred[v], aft, classes, cls, ccol, b, free[j], w, rdy)
            cost = f + alpha * (dmem if j == 0 else 0.0)
            if best_j < 0 or cost < best_cost:
                best_j, best_cost, best_f = j, cost, f
        classes[v] = 0 if best_j == 0 else 1
        cores[v] = best_j
        aft[v] = best_f
        free[best_j] = best_f
    latency = engine._plan_latency(graph, mem, b, classes, aft, io_transfers)
    memory = engine.gpu_plan_memory(graph, cm, classes)
    plan = Plan(order=order, selection=tuple(classes), cores=tuple(cores), k_star=k_prime, alpha=alpha)
    return CoreCountPoint(k_prime, plan, latency, memory, latency + alpha * memory)


def sweep_core_counts(
    graph: "Graph", cm: CostModel, order: Order, alpha: float, io_transfers: bool = False
) -> list[CoreCountPoint]:
    """Algorithm 2 for every budget 0..k (one :class:`CoreCountPoint` each)."""
    if alpha < 0:
        raise ValueError(f"alpha must be non-negative, got {alpha}")
    check_compatible(graph, cm)
    tables = (cm.W.tolist(), cm.Mem.tolist(), cm.incoming, float(cm.b), set(graph.entries))
    return [
        _greedy_for_budget(graph, cm, order, alpha, kp, io_transfers, tables)
        for kp in range(cm.k + 1)
    ]


def select_devices(
    graph: "Graph", cm: CostModel, order: Order, alpha: float, io_transfers: bool = False
) -> Plan:
    """Budget with the lowest total cost; the lowest budget wins ties."""
    pts = sweep_core_counts(graph, cm, order, alpha, io_transfers)
    win = pts[0]
    for p in pts[1:]:
        if p.total_cost < win.total_cost:
            win = p
    return win.plan


def latency_optimal_plan(graph: "Graph", cm: CostModel, io_transfers: bool = False) -> Plan:
    """The paper's latency-optimal pattern: hybrid order, alpha = 0."""
    return select_devices(graph, cm, topo_sort_hybrid(graph, cm), 0.0, io_transfers)


@dataclass(frozen=True)
class AlphaPoint:
    alpha: float
    plan: Plan
    latency: float
    gpu_memory: float
    k_star: int


def _alpha_grid(spec: str) -> list[float]:
    """``start:stop:step`` inclusive grid, computed as ``start + i*step`` to
    avoid drift (the CLI's default is ``0:1:0.1``, reference cli.py:125-140)."""
    lo, hi, step = (float(x) for x in spec.split(":"))
    if step <= 0 or hi < lo or lo < 0:
        raise ValueError(f"bad alpha range {spec!r}")
    count = int((hi - lo) / step + 1e-9) + 1
    return [lo + i * step for i in range(count)]


def sweep_alpha(
    graph: "Graph", cm: CostModel, alphas="0:1:0.1", io_transfers: bool = False
) -> list[AlphaPoint]:
    """Latency/memory frontier: one greedy plan per alpha, each re-evaluated
    with :func:`engine.evaluate` (the rows of the reference's ``sweep``)."""
    grid = _alpha_grid(alphas) if isinstance(alphas, str) else [float(a) for a in alphas]
    order = topo_sort_hybrid(graph, cm)
    out = []
    for a in grid:
        plan = select_devices(graph, cm, order, a, io_transfers)
        ev = engine.evaluate(graph, cm, plan, io_transfers)
        out.append(AlphaPoint(a, plan, ev.latency, ev.gpu_memory, plan.k_star))
    return out


def sweep_csv(graph: "Graph", cm: CostModel, alphas="0:1:0.1", io_transfers: bool = False) -> str:
    """The frontier as the reference's ``sweep.csv`` text (cli.py:259-306):
    ``kind,alpha,latency_ms,gpu_memory_mb,k_star`` — one ``plan`` row per alpha,
    then the all-GPU and all-CPU baselines; floats written with ``repr``."""
    lines = ["kind,alpha,latency_ms,gpu_memory_mb,k_star"]
    for p in sweep_alpha(graph, cm, alphas, io_transfers):
        lines.append(f"plan,{p.alpha!r},{p.latency!r},{p.gpu_memory!r},{p.k_star}")
    gpu_plan, cpu_plan = engine.baseline_plans(graph, cm, io_transfers)
    for kind, plan, k in (("baseline-gpu", gpu_plan, 0), ("baseline-cpu", cpu_plan, cpu_plan.k_star)):
        ev = engine.evaluate(graph, cm, plan, io_transfers)
        lines.append(f"{kind},,{ev.latency!r},{ev.gpu_memory!r},{k}")
    return "\n".join(lines) + "\n"


def memory_optimal_alpha(
    graph: "Graph",
    cm: CostModel,
    slo_ms: float | None = None,
    alphas="0:1:0.1",
    io_transfers: bool = False,
) -> AlphaPoint:
    """Memory-optimal pattern: among the frontier points whose latency meets
    the SLO, the one with the least GPU memory (largest alpha on ties).

    The default SLO is the all-GPU pattern's latency ("without exceeding the
    GPU execution pattern").  If no point meets it the
    latency-optimal (alpha=0) point is returned.
    """
    if slo_ms is None:
        gpu_plan, _ = engine.baseline_plans(graph, cm, io_transfers)
        slo_ms = engine.evaluate(graph, cm, gpu_plan, io_transfers).latency
    pts = sweep_alpha(graph, cm, alphas, io_transfers)
    feasible = [p for p in pts if p.latency <= slo_ms]
    if not feasible:
        return pts[0]
    best = feasible[0]
    for p in feasible[1:]:
        if p.gpu_memory <= best.gpu_memory:
            best = p
    return best


def crossing_count(graph: "Graph", selection) -> int:
    """Edges whose endpoints sit on opposite sides of the PCIe link."""
    return sum((selection[s] == 0) != (selection[d] == 0) for s, d in graph.edge_set)


def reduce_movements(
    graph: "Graph", cm: CostModel, plan: Plan, threshold: int | None = None, io_transfers: bool = False
) -> Plan:
    """Flip 'lonely' nodes (all children, or all predecessors, on the other
    side) while the objective does not increase, until the crossing count
    is at most ``threshold`` (default ``max(1, n // 10)``), a full scan
    changes nothing, or a scan would restart from an assignment already seen
    (where the reference, planner.py:303-356, never terminates)."""
    check_compatible(graph, cm)
    if threshold is None:
        threshold = max(1, graph.n // 10)
    if threshold < 0:
        raise ValueError(f"threshold must be non-negative, got {threshold}")
    cls = list(plan.selection)
    cur_plan = plan
    cur_obj = engine.evaluate(graph, cm, plan, io_transfers).objective
    pred, succ = graph.pred, graph.succ
    visited: set[tuple[int, ...]] = set()
    while crossing_count(graph, cls) > threshold:
        # The reference loops forever when equal-objective flips cycle (e.g.
        # gen_lstm_grid(2, 4) with the cpu-comparable preset); a scan that
        # starts from an already-seen assignment would repeat that cycle, so
        # stop there.  Terminating runs never revisit a state: identical plans.
        state = tuple(cls)
        if state in visited:
            break
        visited.add(state)
        progressed = False
        for v in range(graph.n):
            mine = cls[v]
            alone_out = bool(succ[v]) and all(cls[s] != mine for s in succ[v])
            alone_in = bool(pred[v]) and all(cls[m] != mine for m in pred[v])
            if not (alone_out or alone_in):
                continue
            if mine == 0 and plan.k_star < 1:
                continue
            trial = cls.copy()
            trial[v] = 1 - mine
            cores, _aft, _lat = engine.resolve_cores(
                graph, cm, plan.order.seq, trial, plan.k_star, io_transfers
            )
            cand = replace(cur_plan, selection=tuple(trial), cores=tuple(cores))
            obj = engine.evaluate(graph, cm, cand, io_transfers).objective
            if obj <= cur_obj:
                cls, cur_plan, cur_obj = trial, cand, obj
                progressed = True
        if not progressed:
            break
    return cur_plan


def check_plan(graph: "Graph", cm: CostModel, plan: Plan) -> None:
    engine._check_plan_shape(graph, cm, plan)
    if plan.k_star == 0 and any(c != 0 for c in plan.selection):
        raise ValueError("k_star is 0 but the plan places nodes on the CPU")
    if plan.alpha < 0:
        raise ValueError(f"alpha must be non-negative, got {plan.alpha}")


def save_plan(plan: Plan, path) -> None:
    doc = {
        "order": list(plan.order.seq),
        "selection": list(plan.selection),
        "cores": list(plan.cores),
        "k_star": plan.k_star,
        "alpha": plan.alpha,
    }
    Path(path).write_text(json.dumps(doc, indent=2) + "\n")


def load_plan(path) -> Plan:
    try:
        doc = json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise PlanFormatError(f"{path}: not valid JSON: {exc}") from exc
    if not isinstance(doc, dict):
        raise PlanFormatError(f"{path}: expected a JSON object")
    for key in ("order", "selection", "cores", "k_star", "alpha"):
        if key not in doc:
            raise PlanFormatError(f"{path}: missing key {key!r}")
    lists = {k: doc[k] for k in ("order", "selection", "cores")}
    for name, seq in lists.items():
        if not isinstance(seq, list) or any(not isinstance(x, int) for x in seq):
            raise PlanFormatError(f"{path}: {name} must be a list of integers")
    if len({len(v) for v in lists.values()}) != 1:
        raise PlanFormatError(f"{path}: order/selection/cores lengths differ")
    k_star, alpha = doc["k_star"], doc["alpha"]
    if not isinstance(k_star, int) or k_star < 0:
        raise PlanFormatError(f"{path}: k_star must be a non-negative integer")
    if not isinstance(alpha, (int, float)) or alpha < 0:
        raise PlanFormatError(f"{path}: alpha must be a non-negative number")
    if any(s not in (0, 1) for s in lists["selection"]):
        raise PlanFormatError(f"{path}: selection entries must be 0 or 1")
    return Plan(
        order=Order(seq=tuple(lists["order"])),
        selection=tuple(lists["selection"]),
        cores=tuple(lists["cores"]),
        k_star=k_star,
        alpha=float(alpha),
    )
