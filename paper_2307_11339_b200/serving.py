"""Multi-model serving on one B200: residency, LRU/FIFO eviction, swaps, SLOs.

Two layers, one accounting:

* The reference's serving study, restated with the same API and the same
  arithmetic (``hetsched.servingsim``, /root/reference/pkg/src/hetsched/
  servingsim.py): ``ModelEntry`` 45-54, ``Workload`` 57-71, ``Event`` /
  ``ServingMetrics`` / ``ServingResult`` 74-100, the LRU/FIFO policies
  103-128, ``run_serving`` 143-237, ``compare_patterns`` 259-288,
  ``slo_from_latency`` 291-295, ``events_to_csv`` 298-302 and the scenario
  files 305-427.  It consumes scalar per-model latencies, footprints and
  weight sizes, and its event log is bit-identical to the reference's
  (``tests/test_serving_golden.py`` against fixtures the reference wrote).
* :class:`ResidencyServer`, the same loop over REAL models: each model is an
  :class:`~.rnn.RNNExecutor` whose packed weights live in pinned host memory
  while it is not resident; a request for a non-resident model evicts
  residents by the same policy until its measured HBM footprint fits, uploads
  its packed weights (the swap), then runs the request's forward through
  ``hs_rnn_forward_host``.  Load and execution times are CUDA-event
  measurements, not ``weights_mb / b`` and a profile scalar; they are placed on
  the reference's virtual request clock (arrival, wait, stall, execution), so
  the measured run and :func:`run_serving` over the measured scalars can be
  compared event by event (``tools/serving_report.py``).

Divergence (documented): eviction frees device memory and costs what the
free measures (microseconds) — the weights are immutable and the host master
copy stays, so there is no offload transfer; the reference charges
``weights_mb / b`` for it (servingsim.py:201-209).
"""
from __future__ import annotations

import json
import statistics
import time
from collections import OrderedDict
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable

import numpy as np

__all__ = [
    "ModelEntry", "Workload", "Scenario", "ScenarioError", "Event", "ServingMetrics", "ServingResult",
    "PatternReport", "run_serving", "compare_patterns", "slo_from_latency", "events_to_csv", "save_scenario",
    "load_scenario", "SLO_SLACK", "POLICIES", "ResidencyServer", "MeasuredRequest",
]

#: Default SLO slack over a model's reference latency (servingsim.py:37-38).
SLO_SLACK = 1.25


class ScenarioError(ValueError):
    """An inconsistent serving scenario (servingsim.py:41-42)."""


@dataclass(frozen=True)
class ModelEntry:
    """One deployable model: HBM footprint while resident, per-request
    latency, weight bytes moved by a load, and its latency target (MB, ms)."""

    id: str
    gpu_footprint_mb: float
    exec_latency_ms: float
    weights_mb: float
    slo_ms: float


@dataclass(frozen=True)
class Workload:
    """Request stream: ``uniform`` = round robin over the models, ``random`` =
    seeded uniform choice per request.  ``interarrival_ms`` 0 is closed loop
    (each request arrives when the server frees up); > 0 spaces arrivals
    evenly so queueing builds up."""

    total_requests: int
    pattern: str = "uniform"
    seed: int = 0
    interarrival_ms: float = 0.0


@dataclass(frozen=True)
class Event:
    t: float
    event: str
    model: str
    detail: str


@dataclass(frozen=True)
class ServingMetrics:
    invocations: int
    violations: int
    swaps: int

    @property
    def slo_violation(self) -> float:  # PAPER.md Eq. (7)
        return self.violations / self.invocations

    @property
    def swapping_rate(self) -> float:  # PAPER.md Eq. (8)
        return self.swaps / self.invocations


@dataclass(frozen=True)
class ServingResult:
    metrics: ServingMetrics
    events: tuple[Event, ...]


class _Recency:
    """LRU: the victim is the model touched longest ago."""

    def __init__(self):
        self._q: OrderedDict[str, None] = OrderedDict()

    def touch(self, mid: str) -> None:
        self._q.pop(mid, None)
        self._q[mid] = None

    def drop(self, mid: str) -> None:
        self._q.pop(mid, None)

    def victim(self) -> str:
        return next(iter(self._q))


class _Arrival(_Recency):
    """FIFO: the victim is the model loaded earliest; later touches do not count."""

    def touch(self, mid: str) -> None:
        if mid not in self._q:
            self._q[mid] = None


POLICIES = {"lru": _Recency, "fifo": _Arrival}


def _sequence(n_models: int, workload: Workload) -> Iterable[int]:
    """Model index of each request (servingsim.py:131-140)."""
    if workload.pattern == "uniform":
        return (r % n_models for r in range(workload.total_requests))
    if workload.pattern == "random":
        rng = np.random.default_rng(workload.seed)
        return (int(rng.integers(0, n_models)) for _ in range(workload.total_requests))
    raise ScenarioError(f"unknown workload pattern {workload.pattern!r}")


def _validate(models, capacity_mb, workload, bandwidth_mb_per_ms, policy):
    if not models:
        raise ScenarioError("scenario has no models")
    ids = [m.id for m in models]
    if len(set(ids)) != len(ids):
        raise ScenarioError("model ids must be unique")
    if capacity_mb <= 0:
        raise ScenarioError(f"capacity must be positive, got {capacity_mb}")
    if bandwidth_mb_per_ms is not None and bandwidth_mb_per_ms <= 0:
        raise ScenarioError(f"bandwidth must be positive, got {bandwidth_mb_per_ms}")
    if workload.total_requests < 1:
        raise ScenarioError("workload needs at least one request")
    if workload.interarrival_ms < 0:
        raise ScenarioError("interarrival time cannot be negative")
    for m in models:
        if m.gpu_footprint_mb > capacity_mb:
            raise ScenarioError(f"model {m.id} footprint {m.gpu_footprint_mb} MB exceeds capacity {capacity_mb} MB")
        if m.slo_ms <= 0:
            raise ScenarioError(f"model {m.id} has a non-positive SLO")
    if policy not in POLICIES:
        raise ScenarioError(f"unknown eviction policy {policy!r}")


class _Loop:
    """The per-request accounting shared by the simulated and the measured
    server (servingsim.py:189-232): arrival, start = max(arrival, free),
    evictions until the model fits, load, execution, SLO check.  The caller
    supplies the stall and execution times; the float expression order is
    the reference's, so simulated event logs are bit-identical."""

    def __init__(self, models, capacity_mb, workload, policy):
        self.models = list(models)
        self.by_id = {m.id: m for m in self.models}
        self.capacity = capacity_mb
        self.workload = workload
        self.pol = POLICIES[policy]()
        self.resident: dict[str, float] = {}
        self.used = 0.0
        self.loaded_once: set[str] = set()
        self.events: list[Event] = []
        self.violations = 0
        self.swaps = 0
        self.free_at = 0.0

    def requests(self):
        return enumerate(_sequence(len(self.models), self.workload))

    def begin(self, r: int, m: ModelEntry) -> tuple[float, float]:
        arrival = r * self.workload.interarrival_ms if self.workload.interarrival_ms > 0 else self.free_at
        start = max(arrival, self.free_at)
        self.events.append(Event(t=arrival, event="arrive", model=m.id, detail=""))
        return arrival, start

    def victims(self, m: ModelEntry, start: float, on_evict) -> float:
        """Evict until ``m`` fits; returns the summed eviction stall."""
        stall = 0.0
        while self.used + m.gpu_footprint_mb > self.capacity:
            v = self.pol.victim()
            freed = self.resident.pop(v)
            self.used -= freed
            self.pol.drop(v)
            stall += on_evict(v)
            self.events.append(Event(t=start, event="evict", model=v, detail=f"freed={freed!r}"))
        return stall

    def loaded(self, m: ModelEntry, start: float) -> None:
        kind = "swap" if m.id in self.loaded_once else "cold"
        if kind == "swap":
            self.swaps += 1
        self.loaded_once.add(m.id)
        self.resident[m.id] = m.gpu_footprint_mb
        self.used += m.gpu_footprint_mb
        self.events.append(Event(t=start, event="load", model=m.id, detail=kind))

    def finish(self, m: ModelEntry, arrival: float, start: float, stall: float, exec_ms: float) -> float:
        wait = start - arrival
        latency = wait + stall + exec_ms
        violated = latency > m.slo_ms
        if violated:
            self.violations += 1
        self.free_at = start + stall + exec_ms
        self.events.append(Event(t=self.free_at, event="complete", model=m.id,
                                 detail=f"latency={latency!r},violation={int(violated)}"))
        return latency

    def result(self) -> ServingResult:
        met = ServingMetrics(invocations=self.workload.total_requests, violations=self.violations, swaps=self.swaps)
        return ServingResult(metrics=met, events=tuple(self.events))


def run_serving(models, capacity_mb: float, workload: Workload, bandwidth_mb_per_ms: float = 12.0,
                policy: str = "lru") -> ServingResult:
    """Simulated serving over scalar model entries (servingsim.py:143-237):
    a load stalls ``weights_mb / b`` and so does each victim's offload."""
    models = list(models)
    _validate(models, capacity_mb, workload, bandwidth_mb_per_ms, policy)
    b = bandwidth_mb_per_ms
    loop = _Loop(models, capacity_mb, workload, policy)
    for r, mi in loop.requests():
        m = models[mi]
        arrival, start = loop.begin(r, m)
        stall = 0.0
        if m.id not in loop.resident:
            stall = loop.victims(m, start, lambda v: loop.by_id[v].weights_mb / b)
            stall += m.weights_mb / b
            loop.loaded(m, start)
        loop.pol.touch(m.id)
        loop.finish(m, arrival, start, stall, m.exec_latency_ms)
    return loop.result()


@dataclass(frozen=True)
class PatternReport:
    """Serving metrics of the three deployment patterns side by side
    (servingsim.py:240-256; Table 6)."""

    rows: tuple[tuple[str, ServingResult], ...]

    def metrics(self) -> dict[str, dict]:
        return {
            name: {"invocations": r.metrics.invocations, "violations": r.metrics.violations,
                   "swaps": r.metrics.swaps, "slo_violation": r.metrics.slo_violation,
                   "swapping_rate": r.metrics.swapping_rate}
            for name, r in self.rows
        }


PATTERNS = ("gpu", "latency-optimal", "memory-optimal")


def compare_patterns(models_gpu, models_latopt, models_memopt, capacity_mb: float, workload: Workload,
                     bandwidth_mb_per_ms: float = 12.0, policy: str = "lru") -> PatternReport:
    """One workload over the three variants of the same model list
    (servingsim.py:259-288)."""
    ids = [m.id for m in models_gpu]
    for name, other in (("latency-optimal", models_latopt), ("memory-optimal", models_memopt)):
        if [m.id for m in other] != ids:
            raise ScenarioError(f"{name} variant does not list the same model ids as the gpu variant")
    return PatternReport(rows=tuple(
        (name, run_serving(ms, capacity_mb, workload, bandwidth_mb_per_ms, policy))
        for name, ms in zip(PATTERNS, (models_gpu, models_latopt, models_memopt))))


def slo_from_latency(reference_latency_ms: float, slack: float = SLO_SLACK) -> float:
    """Default latency target: reference latency x slack (servingsim.py:291-295)."""
    if reference_latency_ms <= 0:
        raise ValueError("reference latency must be positive")
    return reference_latency_ms * slack


def events_to_csv(events) -> str:
    rows = ["t,event,model,detail"] + [f"{e.t!r},{e.event},{e.model},{e.detail}" for e in events]
    return "\n".join(rows) + "\n"


# ------------------------------------------------------------------ scenarios

@dataclass(frozen=True)
class Scenario:
    """Capacity, bandwidth, workload and either one model list or one list per
    pattern (servingsim.py:305-319)."""

    capacity_mb: float
    bandwidth_mb_per_ms: float
    workload: Workload
    models: tuple[ModelEntry, ...] | None = None
    patterns: dict | None = None

    def __post_init__(self):
        if (self.models is None) == (self.patterns is None):
            raise ScenarioError("scenario needs exactly one of 'models' or 'patterns'")


_MODEL_KEYS = ("id", "gpu_footprint_mb", "exec_latency_ms", "weights_mb", "slo_ms")
_WORKLOAD_DEFAULTS = (("pattern", str, "uniform"), ("seed", int, 0), ("interarrival_ms", float, 0.0))


def _bad(where: str, what: str):
    return ScenarioError(f"{where}: {what}")


def _model(doc, where: str) -> ModelEntry:
    """One model entry of a scenario file (the five _MODEL_KEYS; numbers >= 0)."""
    if not isinstance(doc, dict):
        raise _bad(where, "model entries must be objects")
    absent = [k for k in _MODEL_KEYS if k not in doc]
    if absent:
        raise _bad(where, f"model entry missing key {absent[0]!r}")
    if not isinstance(doc["id"], str):
        raise _bad(where, "model id must be a string")
    nums = []
    for k in _MODEL_KEYS[1:]:
        v = doc[k]
        if isinstance(v, bool) or not isinstance(v, (int, float)) or v < 0:
            raise _bad(where, f"{k} must be a non-negative number")
        nums.append(float(v))
    return ModelEntry(doc["id"], *nums)


def _model_list(lst, where: str) -> tuple[ModelEntry, ...]:
    if not isinstance(lst, list) or not lst:
        raise _bad(where, "expected a non-empty list of models")
    return tuple(_model(m, f"{where}[{i}]") for i, m in enumerate(lst))


def save_scenario(scenario: Scenario, path) -> None:
    """Write a scenario file (the reference's format, servingsim.py:353-376)."""
    w = scenario.workload
    rows = lambda ms: [{k: getattr(m, k) for k in _MODEL_KEYS} for m in ms]  # noqa: E731
    doc: dict = {
        "capacity_mb": scenario.capacity_mb,
        "bandwidth_mb_per_ms": scenario.bandwidth_mb_per_ms,
        "workload": dict(total_requests=w.total_requests, **{k: getattr(w, k) for k, _, _ in _WORKLOAD_DEFAULTS}),
    }
    if scenario.models is None:
        doc["patterns"] = {name: rows(ms) for name, ms in scenario.patterns.items()}
    else:
        doc["models"] = rows(scenario.models)
    Path(path).write_text(json.dumps(doc, indent=2) + "\n")


def load_scenario(path) -> Scenario:
    """Read a scenario file; any inconsistency raises ScenarioError
    (servingsim.py:379-427)."""
    try:
        doc = json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise _bad(str(path), f"not valid JSON: {exc}") from exc
    if not isinstance(doc, dict):
        raise _bad(str(path), "expected a JSON object")
    for k in ("capacity_mb", "bandwidth_mb_per_ms", "workload"):
        if k not in doc:
            raise _bad(str(path), f"missing key {k!r}")
    wd = doc["workload"]
    if not isinstance(wd, dict) or "total_requests" not in wd:
        raise _bad(str(path), "workload must be an object with total_requests")
    extra = {k: cast(wd.get(k, dflt)) for k, cast, dflt in _WORKLOAD_DEFAULTS}
    workload = Workload(total_requests=int(wd["total_requests"]), **extra)
    if workload.pattern not in ("uniform", "random"):
        raise _bad(str(path), f"unknown workload pattern {workload.pattern!r}")
    has = [k for k in ("models", "patterns") if k in doc]
    if len(has) != 1:
        raise _bad(str(path), "need exactly one of 'models' or 'patterns'")
    models = patterns = None
    if has[0] == "models":
        models = _model_list(doc["models"], f"{path} models")
    else:
        pd = doc["patterns"]
        if not isinstance(pd, dict) or not pd:
            raise _bad(str(path), "patterns must be a non-empty object")
        patterns = {name: _model_list(lst, f"{path} patterns[{name}]") for name, lst in pd.items()}
    return Scenario(float(doc["capacity_mb"]), float(doc["bandwidth_mb_per_ms"]), workload, models, patterns)


# ------------------------------------------------------- real residency server

MB = 1e6  # the reference's unit: MB = 10^6 bytes


@dataclass(frozen=True)
class MeasuredRequest:
    """Measured components of one served request (ms, CUDA events)."""

    index: int
    model: str
    wait_ms: float
    evict_ms: float
    load_ms: float
    exec_ms: float
    latency_ms: float


class ResidencyServer:
    """Serves several real models from one B200 under an HBM budget.

    ``models`` maps a model id to an :class:`~.rnn.RNNExecutor`.  A model's
    footprint is what it holds while resident: packed weights, workspace
    and the :class:`~.serve.RNNServer` staging buffers.  Only models in the
    resident set hold device memory; the rest keep their packed weights in
    pinned host memory.  ``slo_ms`` gives each model's latency target
    (default: :func:`slo_from_latency` of its measured warm latency).
    """

    SLOTS = 2  # request staging sets per resident model (requests here are served one at a time)

    def __init__(self, models: dict, capacity_mb: float, policy: str = "lru", slo_ms: dict | None = None,
                 inputs: dict | None = None):
        import torch

        from .rnn import make_input
        from .serve import RNNServer

        if policy not in POLICIES:
            raise ScenarioError(f"unknown eviction policy {policy!r}")
        self.models = dict(models)
        self.capacity_mb = float(capacity_mb)
        self.policy = policy
        self._RNNServer = RNNServer
        self._servers: dict = {}
        self.inputs = {k: (inputs or {}).get(k, None) for k in self.models}
        for k, ex in self.models.items():
            if self.inputs[k] is None:
                self.inputs[k] = make_input(ex.spec, 1).pin_memory()
        self._ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        self.footprint_mb = {}
        self.weights_mb = {}
        for k, ex in self.models.items():
            st = ex.spec
            state = st.layers * st.dirs * st.batch * st.hidden * 4
            staging = (st.seq * st.batch * st.I * 4 + st.seq * st.batch * st.dirs * st.hidden * 4
                       + state * (2 if st.cell == "lstm" else 1) + 2 * state)
            self.footprint_mb[k] = (ex.packed_bytes() + ex.workspace_bytes() + self.SLOTS * staging) / MB
            self.weights_mb[k] = ex.packed_bytes() / MB
            if self.footprint_mb[k] > self.capacity_mb:
                raise ScenarioError(f"model {k} footprint {self.footprint_mb[k]} MB exceeds capacity {capacity_mb} MB")
        self.slo_ms = dict(slo_ms or {})

    # device-side operations, each timed with CUDA events on the current stream
    def _timed(self, fn) -> float:
        import torch

        st = torch.cuda.current_stream()
        self._ev[0].record(st)
        fn()
        self._ev[1].record(st)
        self._ev[1].synchronize()
        return self._ev[0].elapsed_time(self._ev[1])

    def _evict(self, mid: str) -> float:
        t0 = time.perf_counter()
        self._servers.pop(mid, None)
        self.models[mid].offload()
        return (time.perf_counter() - t0) * 1e3

    def _load(self, mid: str) -> float:
        ex = self.models[mid]

        def go():
            ex.load()
            self._servers[mid] = self._RNNServer(ex, slots=self.SLOTS)

        return self._timed(go)

    def _exec(self, mid: str) -> float:
        from .serve import InferenceRequest

        srv = self._servers[mid]
        return srv.run(InferenceRequest(x=self.inputs[mid])).device_ms

    def offload_all(self) -> None:
        for mid in self.models:
            self._evict(mid)

    def warm_latency(self, mid: str, reps: int = 5) -> float:
        """p50 of ``reps`` warm requests with the model resident (ms)."""
        was = self.models[mid].resident
        if mid not in self._servers:
            self._load(mid)
        self._exec(mid)
        ts = [self._exec(mid) for _ in range(reps)]
        if not was:
            self._evict(mid)
        return statistics.median(ts)

    def load_bandwidth_mb_per_ms(self, mid: str | None = None, reps: int = 3) -> float:
        """Measured H2D load bandwidth of a model's packed weights (MB/ms)."""
        mid = mid or next(iter(self.models))
        ts = []
        for _ in range(reps):
            self._evict(mid)
            ts.append(self._load(mid))
        self._evict(mid)
        return self.weights_mb[mid] / statistics.median(ts)

    def entries(self, exec_ms: dict | None = None) -> list[ModelEntry]:
        """The measured scalars as reference :class:`ModelEntry` rows."""
        out = []
        for k in self.models:
            e = exec_ms[k] if exec_ms else self.warm_latency(k)
            slo = self.slo_ms.get(k) or slo_from_latency(e)
            self.slo_ms[k] = slo
            out.append(ModelEntry(k, self.footprint_mb[k], e, self.weights_mb[k], slo))
        return out

    def serve(self, workload: Workload) -> tuple[ServingResult, list[MeasuredRequest]]:
        """Serve ``workload`` for real, starting from an empty device.
        Accounting as :func:`run_serving`, with measured eviction, load and
        execution times in place of the modelled ones."""
        for k in self.models:
            if k not in self.slo_ms:
                self.slo_ms[k] = slo_from_latency(self.warm_latency(k))
        entries = [ModelEntry(k, self.footprint_mb[k], 0.0, self.weights_mb[k], self.slo_ms[k]) for k in self.models]
        _validate(entries, self.capacity_mb, workload, None, self.policy)
        self.offload_all()
        loop = _Loop(entries, self.capacity_mb, workload, self.policy)
        measured = []
        for r, mi in loop.requests():
            m = entries[mi]
            arrival, start = loop.begin(r, m)
            ev_ms = ld_ms = 0.0
            if m.id not in loop.resident:
                ev_ms = loop.victims(m, start, self._evict)
                ld_ms = self._load(m.id)
                loop.loaded(m, start)
            loop.pol.touch(m.id)
            ex_ms = self._exec(m.id)
            lat = loop.finish(m, arrival, start, ev_ms + ld_ms, ex_ms)
            measured.append(MeasuredRequest(r, m.id, start - arrival, ev_ms, ld_ms, ex_ms, lat))
        return loop.result(), measured
