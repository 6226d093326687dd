"""B200-native executor for Chrion's RNN operator-DAG forward path.

Drop-in for the reference toolkit ``hetsched`` on the hot path: the DAG,
profiling-table, planning and evaluation API keep the reference's names and
semantics (plans are bit-exact), while the two seams that change —
the operator executor (reference ``engine.simulate``) and the per-operator
profiler (reference ``costmodel.synth_profile``) — run on hand-written sm_100a
CUDA kernels behind a C ABI (include/hs_rnn.h).  New entry points:
:func:`execute`, :func:`profile_ops`, :func:`run`, :func:`memory_optimal_alpha`.
"""

__version__ = "0.1.0"

from .costmodel import (
    CostModel,
    PRESETS,
    ProfileFormatError,
    SynthParams,
    check_compatible,
    comm_time,
    crossing,
    exec_time,
    load_profile,
    save_profile,
    synth_profile,
)
from .engine import (
    EvalResult,
    NodeSpan,
    Trace,
    TransferSpan,
    baseline_plans,
    evaluate,
    gpu_plan_memory,
    resolve_cores,
    save_trace,
    simulate,
    trace_to_csv,
)
from .graph import (
    Graph,
    GraphFormatError,
    ValidationReport,
    gen_bilstm_grid,
    gen_demo7,
    gen_lstm_grid,
    gen_random_dag,
    load_graph,
    save_graph,
    validate,
)
from .planner import (
    AlphaPoint,
    CoreCountPoint,
    Order,
    Plan,
    PlanFormatError,
    check_plan,
    crossing_count,
    latency_optimal_plan,
    load_plan,
    memory_optimal_alpha,
    reduce_movements,
    save_plan,
    select_devices,
    sweep_alpha,
    sweep_csv,
    sweep_core_counts,
    topo_sort_bfs,
    topo_sort_dfs,
    topo_sort_hybrid,
)
from .rnn import CONFIGS, RNNExecutor, RNNSpec, init_weights, load_library, make_input
from .executor import ExecResult, HostRNN, build_schedule, execute, measure_link_bandwidth, profile_ops
from .parallel import HostStage, LayerPipeline, PeerPipeline, RequestShard, shard_range, stage_layers
from .serve import InferenceRequest, InferenceResponse, RNNServer, register_model, run

__all__ = [
    "__version__",
    # graph
    "Graph", "GraphFormatError", "ValidationReport", "gen_lstm_grid", "gen_bilstm_grid",
    "gen_demo7", "gen_random_dag", "validate", "load_graph", "save_graph",
    # cost model
    "CostModel", "ProfileFormatError", "SynthParams", "PRESETS", "synth_profile", "exec_time",
    "comm_time", "crossing", "check_compatible", "load_profile", "save_profile",
    # planner
    "Order", "Plan", "PlanFormatError", "CoreCountPoint", "AlphaPoint", "topo_sort_bfs",
    "topo_sort_dfs", "topo_sort_hybrid", "select_devices", "sweep_core_counts", "sweep_alpha", "sweep_csv",
    "memory_optimal_alpha", "latency_optimal_plan", "reduce_movements", "check_plan",
    "crossing_count", "load_plan", "save_plan",
    # evaluation
    "EvalResult", "NodeSpan", "TransferSpan", "Trace", "evaluate", "simulate", "resolve_cores",
    "baseline_plans", "gpu_plan_memory", "trace_to_csv", "save_trace",
    # B200 executor
    "RNNSpec", "CONFIGS", "RNNExecutor", "init_weights", "make_input", "load_library",
    "HostRNN", "ExecResult", "build_schedule", "execute", "profile_ops", "measure_link_bandwidth",
    "InferenceRequest", "InferenceResponse", "RNNServer", "register_model", "run",
    # multi-GPU
    "RequestShard", "LayerPipeline", "PeerPipeline", "HostStage", "shard_range", "stage_layers",
]
