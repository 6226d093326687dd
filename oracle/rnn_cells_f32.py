"""Host-CPU reference of the RNN DAG forward in fp32 torch — BASELINE.md §2.

TEST / BASELINE INFRASTRUCTURE ONLY: imported by ``bench.py`` (the
``--impl reference`` arm and the ``cpu_baseline`` leg) and by ``tests/``, as
the timed host baseline and never on the product path.

BASELINE.md §2 defines the host-CPU reference the B200 numbers are reported
against, because the reference (``hetsched``) has no tensor numerics
(SPEC.md:14, 104):

(a) fused ``torch.nn.LSTM`` / ``torch.nn.GRU`` in fp32 on all host cores (the
    best case), and
(b) Chrion-style per-operator dispatch: the cell DAG of ``gen_lstm_grid``
    (graph.py:207-228) evaluated one cell per dispatch in the planner's order
    ``Plan.order.seq`` (planner.py:53-63) — the order the reference's executor
    replays (engine.py:265-418, per-processor queues drained in plan order).

The cell math is PyTorch's LSTM/GRU (gate rows i,f,g,o / r,z,n; GRU hidden
bias inside r*(.)), the same equations as the float64 oracle ``rnn_ref.py``;
the bench checks (b)'s output against that oracle (max-abs <= 1e-4).
"""
from __future__ import annotations

import torch

__all__ = ["cells_forward_f32", "fused_forward_f32", "plan_order"]


def plan_order(spec, alpha: float = 0.0):
    """Plan.order.seq of the latency-optimal plan (alpha = 0) on the spec's
    DAG with the reference's synthetic ``cpu-comparable`` profile (seed 0).
    Uses the unmodified reference planner from ``baseline/_ref`` when it is
    importable (unidirectional grids), else this package's bit-exact planner
    (which also builds the bidirectional grid)."""
    mod = None
    if spec.dirs == 1:
        try:
            import hetsched as mod  # noqa: F401  (baseline/_ref on sys.path)
            from hetsched import costmodel, graph, planner  # noqa: F401
        except Exception:
            mod = None
    if mod is None:
        import paper_2307_11339_b200 as mod
    g = (mod.graph.gen_lstm_grid(spec.layers, spec.seq) if spec.dirs == 1
         else mod.graph.gen_bilstm_grid(spec.layers, spec.seq))
    cm = mod.costmodel.synth_profile(g, mod.costmodel.PRESETS["cpu-comparable"], 0)
    order = mod.planner.topo_sort_hybrid(g, cm)
    plan = mod.planner.select_devices(g, cm, order, alpha)
    return list(plan.order.seq), getattr(mod, "__name__", "?")


class _Cells:
    """Per layer-direction fp32 weights, transposed once (W^T contiguous)."""

    def __init__(self, weights):
        self.w = [{"ihT": w["w_ih"].float().t().contiguous(), "hhT": w["w_hh"].float().t().contiguous(),
                   "b_ih": w["b_ih"].float().contiguous(), "b_hh": w["b_hh"].float().contiguous()} for w in weights]


def cells_forward_f32(cell: str, x: torch.Tensor, weights, order, dirs: int = 1, h0=None, c0=None, prepared=None):
    """One cell per dispatch in ``order`` (node ids ``(l*dirs + d)*T + t``,
    the reference numbering for dirs = 1).  x [T, B, I] fp32 CPU.  Returns
    (y [T, B, dirs*H], h_n, c_n) like ``torch.nn.LSTM``."""
    cell = cell.lower()
    cw = prepared if prepared is not None else _Cells(weights)
    T, B, _ = x.shape
    LD = len(cw.w)
    L = LD // dirs
    H = cw.w[0]["hhT"].shape[0]
    outs = torch.empty((L, T, B, dirs * H))
    cst = torch.empty((L, dirs, T, B, H)) if cell == "lstm" else None
    zeros = torch.zeros((B, H))
    with torch.no_grad():
        for node in order:
            t = node % T
            ld = node // T
            l, d = divmod(ld, dirs)
            tp = t - 1 if d == 0 else t + 1
            first = tp < 0 or tp >= T
            xin = x[t] if l == 0 else outs[l - 1, t]
            hp = (zeros if h0 is None else h0[ld]) if first else outs[l, tp, :, d * H:(d + 1) * H]
            w = cw.w[ld]
            gx = torch.addmm(w["b_ih"], xin, w["ihT"])
            gh = torch.addmm(w["b_hh"], hp, w["hhT"])
            if cell == "lstm":
                cp = (zeros if c0 is None else c0[ld]) if first else cst[l, d, tp]
                g = gx + gh
                i_, f_, g_, o_ = g.chunk(4, 1)
                c = torch.sigmoid(f_) * cp + torch.sigmoid(i_) * torch.tanh(g_)
                cst[l, d, t] = c
                outs[l, t, :, d * H:(d + 1) * H] = torch.sigmoid(o_) * torch.tanh(c)
            else:
                r = torch.sigmoid(gx[:, :H] + gh[:, :H])
                z = torch.sigmoid(gx[:, H:2 * H] + gh[:, H:2 * H])
                n = torch.tanh(gx[:, 2 * H:] + r * gh[:, 2 * H:])
                outs[l, t, :, d * H:(d + 1) * H] = (1.0 - z) * n + z * hp
    hn = torch.empty((LD, B, H))
    cn = torch.empty((LD, B, H)) if cell == "lstm" else None
    for l in range(L):
        for d in range(dirs):
            tl = T - 1 if d == 0 else 0
            hn[l * dirs + d] = outs[l, tl, :, d * H:(d + 1) * H]
            if cn is not None:
                cn[l * dirs + d] = cst[l, d, tl]
    return outs[L - 1], hn, cn


def fused_forward_f32(spec, weights):
    """torch.nn.LSTM / GRU (fp32, CPU) loaded with the same weights."""
    cls = torch.nn.LSTM if spec.cell == "lstm" else torch.nn.GRU
    m = cls(spec.I, spec.hidden, spec.layers, bidirectional=spec.dirs == 2)
    with torch.no_grad():
        for l in range(spec.layers):
            for d in range(spec.dirs):
                sfx = f"_l{l}" + ("_reverse" if d else "")
                w = weights[l * spec.dirs + d]
                getattr(m, "weight_ih" + sfx).copy_(w["w_ih"])
                getattr(m, "weight_hh" + sfx).copy_(w["w_hh"])
                getattr(m, "bias_ih" + sfx).copy_(w["b_ih"])
                getattr(m, "bias_hh" + sfx).copy_(w["b_hh"])
    return m
