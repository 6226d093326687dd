#!/usr/bin/env python
"""Benchmark: LSTM forward seqs/s and p50 latency on B200, with roofline and
host-CPU baseline (BASELINE.json metric).

Workload (N=1 line): config c2 — 2-layer LSTM, hidden 1024, seq 128, batch 64,
fp32 semantics (max-abs 1e-4 vs the float64 oracle), random-init weights,
synthetic inputs.  One step = one forward of the whole layers x timesteps DAG
over one batch.  N GPUs = N independent request shards (batch 64 each, weak
scaling, no collective — the path shards only over independent requests).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W untimed warm-up steps, then exactly K timed steps bracketed by a
barrier + cuda synchronize; L2 is flushed (256 MiB write) before every timed
step, outside the per-step CUDA events; device time = sum of per-step event
durations; the max over ranks is reported.  `e2e` repeats the K steps through
the public request API with pinned host buffers (H2D of x, D2H of y/h_n/c_n
inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LSTM seqs/sec and p50 latency (ms) at 1/2/4/8 B200 vs host-CPU ref; % roofline"
UNIT = "seqs/s"
CONFIG_NAME = "c2"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """SM clocks + throttle reasons during the timed region: NVML every 10 ms
    (plus entry and exit) and nvidia-smi every 200 ms, merged."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        exe = shutil.which("nvidia-smi")
        # NVML readings at entry, every 10 ms and at exit: short timed regions
        # (nvidia-smi's first line can take longer than the region) still get
        # samples under load; nvidia-smi's stream is merged in when present
        self._start_nvml()
        if exe:
            self.proc = subprocess.Popen(
                [exe, f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def _start_nvml(self):
        """No nvidia-smi binary on PATH: the same fields through NVML (nvidia_ml_py)."""
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            return
        bits = [getattr(nv, n, 0) for n in ("nvmlClocksEventReasonHwSlowdown", "nvmlClocksEventReasonHwThermalSlowdown",
                                            "nvmlClocksEventReasonSwThermalSlowdown", "nvmlClocksEventReasonSwPowerCap")]
        self._stop = threading.Event()

        def sample():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            except Exception:
                return
            try:
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                r = 0
            self.samples.append([str(sm), str(mx)] + ["Active" if (b and r & b) else "Not Active" for b in bits])

        def poll():
            while not self._stop.wait(0.01):
                sample()

        sample()  # at entry, after the warm-up: the clocks the timed region starts at

        self._sample = sample  # also taken on exit: short timed regions still get a reading under load

        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()

    def __exit__(self, *exc):
        if getattr(self, "_stop", None) is not None:
            self._sample()
            self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_info():
    import torch

    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "model": model,
            "torch_threads": torch.get_num_threads()}


def spec_name(spec) -> str:
    from paper_2307_11339_b200.rnn import CONFIGS

    for k, v in CONFIGS.items():
        if (v.cell, v.layers, v.hidden, v.seq, v.dirs) == (spec.cell, spec.layers, spec.hidden, spec.seq, spec.dirs):
            return k
    return "custom"


def ref_sample_spec(spec, sample_batch: int, sample_seq: int):
    """The bounded CPU sample of the workload: the first ``sample_batch``
    sequences (and, for long configs, the first ``sample_seq`` timesteps)."""
    return spec.with_(batch=min(spec.batch, sample_batch), seq=min(spec.seq, sample_seq or spec.seq), algo="auto")


class HostReference:
    """BASELINE.md §2 host-CPU path on the sample: fp32 torch, all host
    threads; (b) cell-by-cell in Plan.order (Chrion-style per-operator
    dispatch, oracle/rnn_cells_f32.py) is the timed reference, (a) fused
    torch.nn.LSTM/GRU is reported beside it."""

    def __init__(self, spec, sample_batch: int, sample_seq: int):
        import torch

        from oracle.rnn_cells_f32 import _Cells, fused_forward_f32, plan_order
        from paper_2307_11339_b200 import init_weights, make_input

        reference_planner()  # baseline/_ref on sys.path: the reference planner orders the cells
        self.threads = len(os.sched_getaffinity(0))
        torch.set_num_threads(self.threads)
        self.full = spec
        self.spec = ref_sample_spec(spec, sample_batch, sample_seq)
        self.weights = init_weights(spec, 0)
        self.x = make_input(spec, 1)[: self.spec.seq, : self.spec.batch].contiguous()
        self.order, self.planner_src = plan_order(self.spec)
        self.cells = _Cells(self.weights)
        self.fused = fused_forward_f32(self.spec, self.weights)
        # seqs/s at the FULL sequence length: a T-prefix sample scales by T / sample_seq
        self.seq_scale = self.spec.seq / spec.seq

    def step(self):
        from oracle.rnn_cells_f32 import cells_forward_f32

        return cells_forward_f32(self.spec.cell, self.x, None, self.order, dirs=self.spec.dirs, prepared=self.cells)

    def time_fused(self, reps=3):
        import torch

        with torch.no_grad():
            self.fused(self.x)
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                self.fused(self.x)
                ts.append(time.perf_counter() - t0)
        p50 = statistics.median(ts)
        return {"value": self.spec.batch * self.seq_scale / p50, "p50_ms": p50 * 1e3, "threads": self.threads,
                "what": "fused torch.nn.%s fp32 (best-case host path)" % ("LSTM" if self.spec.cell == "lstm" else "GRU")}

    def check(self, out):
        """max-abs of the timed path's output against the float64 oracle."""
        import numpy as np

        from oracle.rnn_ref import rnn_forward_ref

        ref = rnn_forward_ref(self.spec.cell, self.x.double().numpy(),
                              [{k: v.double().numpy() for k, v in d.items()} for d in self.weights], dirs=self.spec.dirs)
        return max(float(np.abs(o.double().numpy() - r).max()) for o, r in zip(out, ref) if r is not None)

    def describe(self):
        s, f = self.spec, self.full
        part = f"{s.batch} of {f.batch} sequences" + (f", first {s.seq} of {f.seq} timesteps (value scaled to T={f.seq})"
                                                       if s.seq < f.seq else f", full T={f.seq}")
        return (f"{spec_name(f)} cell DAG ({s.layers * s.dirs * s.seq} cells) in Plan.order of the latency-optimal plan "
                f"({self.planner_src} planner, cpu-comparable profile), one torch fp32 dispatch per cell, "
                f"{self.threads} threads; {part}")


def time_cpu_baseline(spec, budget_s: float, sample_batch: int, sample_seq: int = 0):
    """The host reference (HostReference) on the host cores, bounded to ~budget_s seconds."""
    hr = HostReference(spec, sample_batch, sample_seq)
    t0 = time.perf_counter()
    out = hr.step()  # warm (thread pool)
    first = time.perf_counter() - t0
    reps = max(1, min(20, int(budget_s / max(first, 1e-3))))
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        hr.step()
        times.append(time.perf_counter() - t0)
    p50 = statistics.median(times)
    return {"value": hr.spec.batch * hr.seq_scale / p50, "unit": UNIT, "p50_ms": p50 * 1e3, "reps": reps,
            "cores": hr.threads, "sample": hr.describe() + f", median of {reps}",
            "max_abs_vs_f64_oracle": hr.check(out), "torch_fused_fp32": hr.time_fused()}


def time_planner(mod, spec, reps=3):
    """Planner leg of the path on the spec's grid:
    gen_lstm_grid + synth_profile(cpu-comparable, seed 0) + topo_sort_hybrid +
    select_devices(alpha=0) + evaluate + simulate, median ms over ``reps``."""
    graph, costmodel, planner, engine = mod.graph, mod.costmodel, mod.planner, mod.engine
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        g = graph.gen_lstm_grid(spec.layers, spec.seq)
        cm = costmodel.synth_profile(g, costmodel.PRESETS["cpu-comparable"], 0)
        order = planner.topo_sort_hybrid(g, cm)
        plan = planner.select_devices(g, cm, order, 0.0)
        ev = engine.evaluate(g, cm, plan)
        tr = engine.simulate(g, cm, plan)
        ts.append((time.perf_counter() - t0) * 1e3)
    return {"ms": statistics.median(ts), "latency_ms": ev.latency, "makespan_ms": tr.makespan, "k_star": plan.k_star,
            "n": g.n}


def reference_planner():
    """The unmodified reference package from baseline/_ref (None if absent)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "hetsched").exists():
        return None
    sys.path.insert(0, str(ref))
    try:
        import hetsched
        from hetsched import costmodel, engine, graph, planner  # noqa: F401

        return hetsched
    except Exception:
        return None


def roofline_entry(spec, plan, algo, rec_f, rec_ms, gemm_ms, peaks, traffic, sm_mhz=None, sms=148, l2_peak=None,
                   p_ffma_measured=None):
    """Roofline of the dominant kernel, the recurrence: t_roof = max(FLOPs /
    tensor peak, bytes / HBM bandwidth), so frac = max of the two fractions and
    `bound` names the larger.  FLOPs: the algorithmic recurrent FLOPs.  Bytes:
    the W_hh bytes that must cross the memory system — zero when W_hh stays
    resident in shared memory; when it is streamed (plan w_ring > 0, e.g. c4)
    every step of every batch slice re-reads it (4 B/weight in fp32 mode as
    fp16 hi+lo, 2 B in bf16 mode) — plus the xproj reads and y writes."""
    common = {"kernel": f"recurrent wavefront ({algo})", "kernel_ms_per_forward": rec_ms,
              "gemm_ms_per_forward": gemm_ms, "traffic": traffic}
    sec = rec_ms / 1e3
    tf = rec_f / sec / 1e12
    f_tensor = tf / peaks["bf16_tflops"]
    G, H, B, T = spec.G, spec.hidden, spec.batch, spec.seq
    wbytes = (2.0 if spec.dtype == "bf16" else 4.0) * G * H * H
    slices = max(1, plan.get("batch_slices", 1))
    LD = spec.layers * spec.dirs
    # HBM: xproj read + y write per step, and W_hh once per launch when it is
    # streamed (ncu, profiles/r02_summary.md: the W ring's per-step re-reads
    # hit L2 — c4 99.8% of 34 GB of evict_last sectors — so they are L2, not
    # HBM, traffic; see the "l2" entry below)
    streamed = bool(plan.get("w_ring"))
    nbytes = T * LD * (4.0 * B * G * H + 4.0 * B * H) + (wbytes * slices * LD if streamed else 0.0)
    gbs = nbytes / sec / 1e9
    f_hbm = gbs / peaks["hbm_gbs"]
    tensor = dict(achieved=tf, peak=peaks["bf16_tflops"], unit="TFLOP/s", frac=f_tensor, algorithmic_flops=rec_f,
                  peak_source=f"{peaks['source']} dense bf16 (burst)")
    hbm = dict(achieved=gbs, peak=peaks["hbm_gbs"], unit="GB/s", frac=f_hbm, algorithmic_bytes=nbytes,
               peak_source=f"{peaks['source']} HBM copy")
    if f_hbm > f_tensor:
        out = dict(common, bound="hbm", **hbm, other={"bound": "tensor", **tensor})
    else:
        out = dict(common, bound="tensor", **tensor, other={"bound": "hbm", **hbm})
    if streamed and l2_peak:
        l2b = wbytes * slices * T * LD
        out["l2"] = {"achieved": l2b / sec / 1e9, "peak": l2_peak["gbs"], "unit": "GB/s",
                     "frac": l2b / sec / 1e9 / l2_peak["gbs"], "bytes": l2b,
                     "what": "W_hh ring re-reads, one per step per batch slice (served from L2)",
                     "peak_source": l2_peak["source"]}
    if spec.dtype == "f32" and sm_mhz:
        # SURVEY §8d's K2/K3 roofline for fp32 mode: t_roof = max(F_rec / P_FFMA,
        # streamed W_hh bytes / HBM), P_FFMA = SMs x 128 FP32 lanes x 2 x the SM
        # clock measured under load (no byte term when W_hh is SMEM-resident).
        # The north-star target (recurrent kernel >= 50% of its roofline) is
        # stated against this; the kernel exceeds it because it runs on tcgen05.
        p_ffma = p_ffma_measured or sms * 128 * 2 * sm_mhz * 1e6 / 1e12
        wstream = (wbytes * slices if plan.get("w_ring") else 0.0) * T * spec.layers * spec.dirs
        t_roof = max(rec_f / (p_ffma * 1e12), wstream / (peaks["hbm_gbs"] * 1e9))
        out["survey_fp32_roofline"] = {"t_roof_ms": t_roof * 1e3, "kernel_ms": rec_ms, "frac": t_roof / sec,
                                       "p_ffma_tflops": p_ffma, "sm_mhz": sm_mhz, "sms": sms,
                                       "note": "SURVEY 8d K2 formula; P_FFMA " + (
                                           "measured (tools/peak_probe.py)" if p_ffma_measured else
                                           "from the measured SM clock")}
    return out


def describe(spec) -> str:
    kind = ("bi" if spec.dirs == 2 else "") + spec.cell.upper()
    return f"{spec.layers}-layer {kind} H{spec.hidden} T{spec.seq} B{spec.batch}/GPU {spec.dtype}"


def run_pipeline(args, spec, world, rank, local, dev):
    """Layer pipeline over `world` GPUs: rank g owns
    a contiguous layer range and hands its output to rank g+1 — by default
    as bf16 hi/lo planes copied GPU-to-GPU per chunk of `chunk` steps while
    its last recurrence runs (--handoff peer), or as [chunk, B, H] NCCL
    point-to-point sends between per-chunk stage forwards (--handoff nccl).  One timed step = `inflight` requests
    streamed through the pipeline (default: one per stage, so the pipeline
    is full in steady state); value = sequences/s of the whole pipeline."""
    import torch
    import torch.distributed as dist

    from paper_2307_11339_b200 import init_weights, make_input
    from paper_2307_11339_b200.parallel import LayerPipeline
    from paper_2307_11339_b200.rnn import RNNExecutor

    inflight = args.inflight or max(world, 1)
    weights = init_weights(spec, 0)
    if args.handoff == "peer":
        # whole-sequence stage forwards; output planes copied GPU-to-GPU chunk
        # by chunk (hs_rnn_forward_stage / parallel.PeerPipeline)
        from paper_2307_11339_b200.parallel import PeerPipeline, stage_layers

        l0, l1 = stage_layers(spec.layers, world, rank)
        sspec = spec.with_(layers=l1 - l0, input=spec.I if rank == 0 else spec.hidden)
        pipe = PeerPipeline(RNNExecutor(sspec, weights[l0:l1], device=dev), rank, world, chunk=args.chunk)
        pipe.l0, pipe.l1, pipe.model = l0, l1, pipe.ex
        xs = [make_input(spec, 1 + r).to(dev) for r in range(inflight)] if rank == 0 else [None] * inflight
    else:
        pipe = LayerPipeline(spec, weights, rank, world, args.chunk, lambda sp, w: RNNExecutor(sp, w, device=dev))
        xs = [make_input(spec, 1 + r).pin_memory() for r in range(inflight)] if rank == 0 else [None] * inflight

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[dev.index]) if dist.get_backend() == "nccl" else dist.barrier()

    for _ in range(args.warmup):
        pipe.run_many(xs)
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clocks:
        for i in range(args.steps):
            evs[i][0].record()
            pipe.run_many(xs)
            evs[i][1].record()
        torch.cuda.synchronize(dev)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total = sum(step_ms)
    if world > 1:
        t = torch.tensor([total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    if rank == 0:
        seqs = spec.batch * inflight * args.steps
        line = {
            "metric": METRIC, "value": seqs / (total / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total / args.steps, "p50_ms": statistics.median(step_ms),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if spec.dtype == "f32" else "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}: {describe(spec)}, layer-pipelined", "mode": "pipeline",
                       "stages": world, "stage0_layers": [pipe.l0, pipe.l1] if rank == 0 else None,
                       "chunk": args.chunk, "requests_per_step": inflight, "algo": getattr(pipe.model, "algo", None),
                       "handoff": args.handoff,
                       "parallelism": f"layer pipeline x{world} ("
                                      + ("copy-engine GPU-to-GPU hand-off per chunk of steps, stream-ordered counters"
                                         if args.handoff == "peer" else "NCCL P2P hand-off per chunk")
                                      + ", no collective)"},
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_reference(args, spec):
    """The reference arm: BASELINE.md §2's host-CPU path (fp32 torch,
    cell-by-cell in Plan.order, all host threads) on rank 0; other ranks exit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    info = cpu_info()
    hr = HostReference(spec, args.ref_sample_batch, args.ref_sample_seq)
    for _ in range(args.warmup):
        out = hr.step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = hr.step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = hr.spec.batch * hr.seq_scale * args.steps / total
    p50 = statistics.median(times) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3, "p50_ms": p50,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {describe(spec)} forward; reference-arm step = the host sample below",
                   "batch_per_gpu": spec.batch, "sample_batch": hr.spec.batch, "sample_seq": hr.spec.seq},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": hr.threads, "kind": "port",
                         "sample": hr.describe(), "host": info,
                         "max_abs_vs_f64_oracle": hr.check(out), "tolerance": 1e-4,
                         "torch_fused_fp32": hr.time_fused()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    hs = reference_planner()
    if hs is not None:
        line["reference_planner"] = dict(time_planner(hs, spec), package=f"hetsched {hs.__version__} (baseline/_ref)")
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=CONFIG_NAME)
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--cpu-baseline-seconds", type=float, default=15.0)
    ap.add_argument("--cpu-sample-batch", type=int, default=64)
    ap.add_argument("--ref-sample-batch", type=int, default=64)
    ap.add_argument("--ref-sample-seq", type=int, default=0, help="host sample: timestep prefix (0 = full T)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", choices=["shard", "pipeline"], default="shard",
                    help="shard: N independent request shards (weak scaling); pipeline: layers split over N GPUs")
    ap.add_argument("--chunk", type=int, default=32, help="pipeline mode: timesteps per hand-off chunk")
    ap.add_argument("--handoff", choices=["peer", "nccl"], default="peer",
                    help="pipeline mode: peer = one stage forward per request with copy-engine GPU-to-GPU hand-off "
                         "(hs_rnn_forward_stage); nccl = per-chunk stage forwards with NCCL isend/irecv (round 1)")
    ap.add_argument("--inflight", type=int, default=0, help="pipeline mode: requests per timed step (default N)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="shard mode: split this many sequences over the N ranks (parallel.RequestShard, strong "
                         "scaling; BASELINE c5 is batch 256 over 8 B200) instead of the config's batch per GPU")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    from paper_2307_11339_b200.rnn import CONFIGS

    spec = CONFIGS[args.config].with_(algo=args.algo)
    if args.impl == "reference":
        return run_reference(args, spec)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HS_BENCH_ONE_DEVICE=1 (+ HS_BENCH_BACKEND=gloo): every rank on cuda:0 — a
    # code-path check of the multi-rank bench on a one-GPU box, not a measurement
    one_dev = os.environ.get("HS_BENCH_ONE_DEVICE") == "1"
    gpu = 0 if one_dev else local
    if world > 1:
        torch.cuda.set_device(gpu)
        backend = os.environ.get("HS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{gpu}"))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device(f"cuda:{gpu if world > 1 else 0}")
    if args.mode == "pipeline":
        return run_pipeline(args, spec, world, rank, local, dev)

    from paper_2307_11339_b200 import init_weights, make_input
    from paper_2307_11339_b200.parallel import shard_range
    from paper_2307_11339_b200.rnn import RNNExecutor
    from paper_2307_11339_b200.serve import InferenceRequest, RNNServer

    strong = args.global_batch > 0
    if strong:
        # this rank's contiguous slice of a global batch (RequestShard's split);
        # ranks with no sequences are not supported by the timing below
        _start, count = shard_range(args.global_batch, world, rank)
        if count == 0:
            raise SystemExit(f"--global-batch {args.global_batch} leaves rank {rank} without sequences")
        spec = spec.with_(batch=count)
    weights = init_weights(spec, 0)
    ex = RNNExecutor(spec, weights, device=dev)
    x_host = make_input(spec, 1 + rank).pin_memory()
    x = x_host.to(dev)
    outs = ex.alloc_outputs()
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[dev.index]) if dist.get_backend() == "nccl" else dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        ex.forward(x, out=outs)
    torch.cuda.synchronize(dev)

    # ---- device-timed region: exactly K steps
    step_ms, layer_ms = [], []
    launches = 0  # kernels of this library inside the timed region (hs_rnn_last_launch_count)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            *_, lm = ex.forward(x, out=outs, layer_ms=True)
            evs[i][1].record(stream)
            layer_ms.append(lm)
            launches += ex.last_launch_count()
        torch.cuda.synchronize(dev)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = max_over_ranks(sum(step_ms))

    # ---- end-to-end through the public request API (pinned host buffers):
    # a stream of K requests through RNNServer.run_stream — every request's
    # H2D of x and D2H of y/h_n/c_n inside the timed region; request i+1's
    # upload overlaps request i's compute (two staging slots)
    server = RNNServer(ex, slots=int(os.environ.get("HS_STREAM_SLOTS", "3")))
    req = InferenceRequest(x=x_host)
    server.run_stream([req] * 2)
    lat = [server.run(req).device_ms for _ in range(5)]  # single-request latency (sync)
    barrier()
    torch.cuda.synchronize(dev)
    summary = server.run_stream([req] * args.steps)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_total = max_over_ranks(summary.device_ms)
    h2d = summary.h2d_bytes // args.steps
    d2h = summary.d2h_bytes // args.steps
    e2e_ms = lat

    if rank != 0:
        dist.destroy_process_group()
        return 0

    B_total = args.global_batch if strong else spec.batch * world
    value = B_total * args.steps / (total_ms / 1e3)
    p50 = statistics.median(step_ms)
    p90 = sorted(step_ms)[int(0.9 * (len(step_ms) - 1))]
    gemm_f, rec_f = spec.flops()
    rec_ms = statistics.mean(sum(l[1] for l in lm) for lm in layer_ms)  # all layers, per forward
    gemm_ms = statistics.mean(sum(l[0] for l in lm) for lm in layer_ms)
    peaks = load_peaks()
    plan = ex.plan()
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    l2_peak = p_ffma = None
    if tfile.exists():
        tdoc = json.loads(tfile.read_text())
        traffic = tdoc.get(f"{args.config}:{ex.algo}:recurrent")
        l2_peak = tdoc.get("_l2_peak")
    pfile = ROOT / "profiles" / "peaks_fp32_l2.json"  # tools/peak_probe.py on a B200 of this pool
    if pfile.exists():
        pdoc = json.loads(pfile.read_text())
        l2_peak = {"gbs": pdoc["l2_read_gbs_64MiB"],
                   "source": "measured L2 read of a 64 MiB L2-resident buffer (profiles/peaks_fp32_l2.json)"}
        p_ffma = pdoc["ffma_tflops"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "p50_ms": p50, "p90_ms": p90,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f32" if spec.dtype == "f32" else "bf16", "data": "synthetic",
        "config": {"workload": f"{args.config}: {describe(spec)} forward (layers x timesteps DAG)"
                               + (f", global batch {B_total} split over {world} GPU(s)" if strong else ""),
                   "batch_per_gpu": spec.batch, "global_batch": B_total, "algo": ex.algo,
                   "parallelism": f"request-sharded x{world} (no collective)"
                                  + (" (parallel.RequestShard split of one global batch)" if strong else ""), "l2": "flushed (256 MiB write) before each timed step",
                   "e2e_l2": "no flush; per-request working set (2 x 128 MiB xproj + 32 MiB x + 32 MiB y) exceeds the 126 MB L2"},
        "roofline": roofline_entry(spec, plan, ex.algo, rec_f, rec_ms, gemm_ms, peaks, traffic,
                                   sm_mhz=clocks.summary().get("sm_mhz"),
                                   sms=torch.cuda.get_device_properties(dev).multi_processor_count, l2_peak=l2_peak,
                                   p_ffma_measured=p_ffma),
        "plan": plan,
        "e2e": {"value": B_total * args.steps / (e2e_total / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / args.steps,
                "single_request_p50_ms": statistics.median(e2e_ms),
                "api": "RNNServer.run_stream (hs_rnn_forward_host), pinned host x in / y,h_n,c_n out every step"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if world == 1:
        import paper_2307_11339_b200 as pkg

        line["planner"] = dict(time_planner(pkg, spec), note="this package's planner (bit-exact with the reference)")
    if world == 1 and not args.no_cpu_baseline:
        cb = time_cpu_baseline(spec, args.cpu_baseline_seconds, args.cpu_sample_batch, args.ref_sample_seq)
        line["cpu_baseline"] = {"value": cb["value"], "unit": UNIT, "cores": cb["cores"], "kind": "port",
                                "sample": cb["sample"], "p50_ms": cb["p50_ms"], "host": cpu_info(),
                                "max_abs_vs_f64_oracle": cb["max_abs_vs_f64_oracle"],
                                "torch_fused_fp32": cb["torch_fused_fp32"]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
