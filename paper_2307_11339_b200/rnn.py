"""RNN model spec, synthetic weights, and the ctypes binding of libhsrnn.so.

This is the host side of the drop-in boundary (include/hs_rnn.h).  PyTorch
provides device memory and streams; every byte of compute runs in the
library's sm_100a kernels.  There is no CPU fallback: if the library is
missing or no sm_100 device is visible, :func:`load_library` and
:class:`RNNExecutor` raise.

Synthetic data follows SURVEY §8(d): weights ~ U(-1/sqrt(H), 1/sqrt(H)) (the
``nn.LSTM/GRU.reset_parameters`` default) drawn on CPU from
``torch.Generator().manual_seed(seed)``; inputs ~ U(-1, 1) with seed 1.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, replace
from pathlib import Path

import torch

from . import build as _build

__all__ = [
    "RNNSpec",
    "CONFIGS",
    "HsRnnError",
    "load_library",
    "init_weights",
    "make_input",
    "RNNExecutor",
    "ABI_SYMBOLS",
]

CELLS = {"lstm": 0, "gru": 1}
DTYPES = {"f32": 0, "bf16": 1}
ALGOS = {"auto": 0, "simt": 1, "tc": 2}
ALGO_NAMES = {1: "simt", 2: "tc"}
GATES = {"lstm": 4, "gru": 3}

#: every symbol declared in include/hs_rnn.h
ABI_SYMBOLS = (
    "hs_abi_version",
    "hs_last_error",
    "hs_rnn_last_launch_count",
    "hs_rnn_resolve_algo",
    "hs_rnn_plan",
    "hs_rnn_workspace",
    "hs_rnn_packed_size",
    "hs_rnn_pack_weights",
    "hs_rnn_forward_packed",
    "hs_rnn_profile_cells",
    "hs_rnn_forward",
    "hs_rnn_forward_host",
    "hs_rnn_forward_stage",
    "hs_pipeline_export",
    "hs_pipeline_import",
    "hs_pipeline_release",
    "hs_rnn_outputs_ready",
    "hs_rnn_run_cells",
)


class HsRnnError(RuntimeError):
    """A libhsrnn.so call returned a non-zero status."""

    def __init__(self, func: str, code: int, msg: str):
        super().__init__(f"{func} failed (status {code}): {msg}")
        self.code = code


@dataclass(frozen=True)
class RNNSpec:
    """Shape of a stacked (bi)directional LSTM/GRU; ``input`` defaults to H."""

    cell: str
    layers: int
    hidden: int
    seq: int
    batch: int
    input: int | None = None
    dirs: int = 1
    dtype: str = "f32"
    algo: str = "auto"

    def __post_init__(self):
        if self.cell not in CELLS:
            raise ValueError(f"cell must be one of {sorted(CELLS)}, got {self.cell!r}")
        if self.dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}, got {self.dtype!r}")
        if self.algo not in ALGOS:
            raise ValueError(f"algo must be one of {sorted(ALGOS)}, got {self.algo!r}")
        if self.dirs not in (1, 2):
            raise ValueError(f"dirs must be 1 or 2, got {self.dirs}")
        for name in ("layers", "hidden", "seq", "batch"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be positive")

    @property
    def I(self) -> int:
        return self.hidden if self.input is None else self.input

    @property
    def G(self) -> int:
        return GATES[self.cell]

    def layer_input(self, l: int) -> int:
        return self.I if l == 0 else self.dirs * self.hidden

    def with_(self, **kw) -> "RNNSpec":
        return replace(self, **kw)

    def flops(self) -> tuple[float, float]:
        """(input-projection, recurrent) FLOPs of one forward."""
        G, H, T, B = self.G, self.hidden, self.seq, self.batch
        gemm = sum(2.0 * T * B * G * H * self.layer_input(l) for l in range(self.layers)) * self.dirs
        rec = 2.0 * T * B * G * H * H * self.layers * self.dirs
        return gemm, rec


#: BASELINE.json configs c1..c5
CONFIGS: dict[str, RNNSpec] = {
    "c1": RNNSpec("lstm", 1, 128, 16, 1),
    "c2": RNNSpec("lstm", 2, 1024, 128, 64),
    "c3": RNNSpec("gru", 4, 512, 256, 32),
    "c4": RNNSpec("lstm", 8, 2048, 512, 16),
    "c5": RNNSpec("lstm", 3, 1024, 1024, 256, dirs=2, dtype="bf16"),
}


class _Desc(ctypes.Structure):
    _fields_ = [
        ("cell", ctypes.c_int32),
        ("layers", ctypes.c_int32),
        ("dirs", ctypes.c_int32),
        ("input", ctypes.c_int32),
        ("hidden", ctypes.c_int32),
        ("seq", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("algo", ctypes.c_int32),
        ("upload_chunks", ctypes.c_int32),
        ("async_outputs", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 5),
    ]


class StageLink(ctypes.Structure):
    """``hs_stage_link`` (include/hs_rnn.h): a layer-pipeline stage's input
    and output hand-off (device pointers, monotonic 32-bit counters)."""

    _fields_ = [
        ("x_planes", ctypes.c_void_p),
        ("x_avail", ctypes.c_void_p),
        ("x_base", ctypes.c_uint32),
        ("consumed_value", ctypes.c_uint32),
        ("consumed_peer", ctypes.c_void_p),
        ("y_peer_planes", ctypes.c_void_p),
        ("y_peer_avail", ctypes.c_void_p),
        ("y_base", ctypes.c_uint32),
        ("consumed_wait", ctypes.c_uint32),
        ("consumed", ctypes.c_void_p),
        ("chunks", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 5),
    ]


def make_desc(spec: RNNSpec) -> _Desc:
    return _Desc(
        CELLS[spec.cell], spec.layers, spec.dirs, spec.I, spec.hidden, spec.seq, spec.batch,
        DTYPES[spec.dtype], ALGOS[spec.algo],
    )


_LIB: ctypes.CDLL | None = None


def load_library(path: str | Path | None = None, build_if_missing: bool = False) -> ctypes.CDLL:
    """Load libhsrnn.so (in-tree).  Raises if it is absent — there is no
    fallback implementation."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    # HS_LIB_PATH: a variant build of the same sources (A/B experiments, debug traces)
    lib_path = Path(path) if path else Path(os.environ.get("HS_LIB_PATH") or _build.library_path())
    if not lib_path.exists():
        if build_if_missing:
            lib_path = _build.build()
        else:
            raise RuntimeError(
                f"{lib_path} is missing: build it with `python -m paper_2307_11339_b200.build` "
                "(there is no CPU fallback for the RNN executor)"
            )
    lib = ctypes.CDLL(str(lib_path))
    vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32
    pd = ctypes.POINTER(_Desc)
    pvp = ctypes.POINTER(vp)
    lib.hs_abi_version.restype = ctypes.c_int
    lib.hs_last_error.restype = ctypes.c_char_p
    lib.hs_rnn_last_launch_count.restype = ctypes.c_int
    lib.hs_rnn_resolve_algo.argtypes = [pd, ctypes.POINTER(i32)]
    lib.hs_rnn_workspace.argtypes = [pd, ctypes.POINTER(sz)]
    lib.hs_rnn_plan.argtypes = [pd, ctypes.POINTER(i32)]
    lib.hs_rnn_packed_size.argtypes = [pd, ctypes.POINTER(sz)]
    lib.hs_rnn_pack_weights.argtypes = [pd, pvp, pvp, pvp, pvp, vp, sz, vp]
    lib.hs_rnn_forward_packed.argtypes = [pd, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, ctypes.POINTER(ctypes.c_float)]
    fp = ctypes.POINTER(ctypes.c_float)
    lib.hs_rnn_profile_cells.argtypes = [pd, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, fp, fp]
    lib.hs_rnn_forward.argtypes = [pd, vp, pvp, pvp, pvp, pvp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.hs_rnn_forward_host.argtypes = [pd, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.hs_rnn_forward_stage.argtypes = [pd, vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(StageLink), vp, sz, vp]
    lib.hs_rnn_outputs_ready.argtypes = [vp, vp]
    lib.hs_pipeline_export.argtypes = [vp, vp, ctypes.POINTER(sz)]
    lib.hs_pipeline_import.argtypes = [vp, sz, ctypes.POINTER(vp)]
    lib.hs_pipeline_release.argtypes = [vp]
    lib.hs_rnn_run_cells.argtypes = [pd, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    for name in ABI_SYMBOLS[3:]:
        getattr(lib, name).restype = ctypes.c_int
    if lib.hs_abi_version() != 1:
        raise RuntimeError(f"{lib_path}: ABI version {lib.hs_abi_version()} != 1")
    if path is None:
        _LIB = lib
    return lib


def _check(lib, func: str, code: int) -> None:
    if code != 0:
        raise HsRnnError(func, code, lib.hs_last_error().decode(errors="replace"))


def init_weights(spec: RNNSpec, seed: int = 0) -> list[dict[str, torch.Tensor]]:
    """PyTorch-default init U(-1/sqrt(H), 1/sqrt(H)); CPU fp32 tensors, one dict
    per layer-direction ``l*dirs + d``, drawn in (w_ih, w_hh, b_ih, b_hh) order."""
    gen = torch.Generator().manual_seed(seed)
    bound = 1.0 / math.sqrt(spec.hidden)
    GH = spec.G * spec.hidden
    out = []
    for l in range(spec.layers):
        for _d in range(spec.dirs):
            shapes = {
                "w_ih": (GH, spec.layer_input(l)),
                "w_hh": (GH, spec.hidden),
                "b_ih": (GH,),
                "b_hh": (GH,),
            }
            out.append({k: (torch.rand(s, generator=gen) * 2.0 - 1.0) * bound for k, s in shapes.items()})
    return out


def make_input(spec: RNNSpec, seed: int = 1, batch: int | None = None) -> torch.Tensor:
    """x ~ U(-1, 1), shape [T, B, I], CPU fp32."""
    gen = torch.Generator().manual_seed(seed)
    B = spec.batch if batch is None else batch
    return torch.rand((spec.seq, B, spec.I), generator=gen) * 2.0 - 1.0


def _ptr_array(ts):
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr


class GraphedForward:
    """One captured device forward (``RNNExecutor.graph``): ``x`` is the static
    input buffer, ``y`` / ``h_n`` / ``c_n`` the outputs every replay writes."""

    def __init__(self, g, x, out):
        self.g = g
        self.x = x
        self.y, self.h_n, self.c_n = out

    def replay(self, x: torch.Tensor | None = None):
        """Copy ``x`` (if given) into the static input on the current stream,
        replay the graph, return ``(y, h_n, c_n)`` (the static outputs)."""
        if x is not None:
            if tuple(x.shape) != tuple(self.x.shape):
                raise ValueError(f"x has shape {tuple(x.shape)}, expected {tuple(self.x.shape)}")
            self.x.copy_(x)
        self.g.replay()
        return self.y, self.h_n, self.c_n


class RNNExecutor:
    """A (bi)directional LSTM/GRU resident on one B200.

    Construction copies the weights to the device and repacks them into the
    kernel layout once (``hs_rnn_pack_weights``); :meth:`forward` then runs
    the whole layers x timesteps DAG with the packed weights.
    """

    def __init__(self, spec: RNNSpec, weights, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("RNNExecutor needs a CUDA (sm_100) device; there is no CPU fallback")
        self.spec = spec
        self.lib = load_library()
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        self.desc = make_desc(spec)
        with torch.cuda.device(self.device):
            a = ctypes.c_int32()
            _check(self.lib, "hs_rnn_resolve_algo", self.lib.hs_rnn_resolve_algo(ctypes.byref(self.desc), ctypes.byref(a)))
            self.algo = ALGO_NAMES[a.value]
            n = ctypes.c_size_t()
            _check(self.lib, "hs_rnn_packed_size", self.lib.hs_rnn_packed_size(ctypes.byref(self.desc), ctypes.byref(n)))
            self._packed_n = max(n.value, 1)
            self.packed = torch.empty(self._packed_n, dtype=torch.uint8, device=self.device)
            self._packed_host = None
            _check(self.lib, "hs_rnn_workspace", self.lib.hs_rnn_workspace(ctypes.byref(self.desc), ctypes.byref(n)))
            self._ws_n = max(n.value, 1)
            self.workspace = torch.empty(self._ws_n, dtype=torch.uint8, device=self.device)
            self.weights = [
                {k: v.to(self.device, torch.float32).contiguous() for k, v in w.items()} for w in weights
            ]
            if len(self.weights) != spec.layers * spec.dirs:
                raise ValueError(f"expected {spec.layers * spec.dirs} layer-direction weight sets, got {len(weights)}")
            for ld, w in enumerate(self.weights):
                l = ld // spec.dirs
                GH = spec.G * spec.hidden
                want = {"w_ih": (GH, spec.layer_input(l)), "w_hh": (GH, spec.hidden), "b_ih": (GH,), "b_hh": (GH,)}
                for k, shp in want.items():
                    if tuple(w[k].shape) != shp:
                        raise ValueError(f"layer-direction {ld}: {k} has shape {tuple(w[k].shape)}, expected {shp}")
            stream = torch.cuda.current_stream(self.device)
            arrs = [_ptr_array([w[k] for w in self.weights]) for k in ("w_ih", "w_hh", "b_ih", "b_hh")]
            _check(
                self.lib,
                "hs_rnn_pack_weights",
                self.lib.hs_rnn_pack_weights(
                    ctypes.byref(self.desc), *arrs, self.packed.data_ptr(), self.packed.numel(), stream.cuda_stream
                ),
            )

    # ---------------------------------------------------------------- residency
    # A serving process keeps more models than fit in HBM (servingsim.py:1-8):
    # the packed weights have a pinned host master copy, and a non-resident
    # executor holds no device memory.  Loading is one H2D copy of the packed
    # buffer (weights are immutable, so eviction needs no copy back).

    @property
    def resident(self) -> bool:
        return self.packed is not None

    def packed_bytes(self) -> int:
        return int(self._packed_n)

    def workspace_bytes(self) -> int:
        return int(self._ws_n)

    def offload(self) -> None:
        """Release this model's device memory (packed weights, workspace and
        the fp32 weight copies); a pinned host copy of the packed buffer is
        kept for :meth:`load`."""
        if not self.resident:
            return
        if self._packed_host is None:
            self._packed_host = torch.empty(self.packed.numel(), dtype=torch.uint8).pin_memory()
            self._packed_host.copy_(self.packed)
        if self.weights and self.weights[0]["w_ih"].device.type != "cpu":
            self.weights = [{k: v.cpu() for k, v in w.items()} for w in self.weights]
        self.packed = None
        self.workspace = None

    def load(self, stream=None) -> None:
        """Make the model resident again: allocate its device buffers and
        upload the packed weights (asynchronous on ``stream``, default the
        current stream; later work on that stream is ordered after it)."""
        if self.resident:
            return
        with torch.cuda.device(self.device):
            st = stream if stream is not None else torch.cuda.current_stream(self.device)
            with torch.cuda.stream(st):
                packed = torch.empty(self._packed_n, dtype=torch.uint8, device=self.device)
                packed.copy_(self._packed_host, non_blocking=True)
                self.workspace = torch.empty(self._ws_n, dtype=torch.uint8, device=self.device)
            self.packed = packed

    def _require_resident(self):
        if not self.resident:
            raise RuntimeError("model is not resident on the device (offloaded); call load() first")

    def plan(self) -> dict:
        """The library's execution plan for this model (``hs_rnn_plan``)."""
        info = (ctypes.c_int32 * 8)()
        _check(self.lib, "hs_rnn_plan", self.lib.hs_rnn_plan(ctypes.byref(self.desc), info))
        return {"algo": ALGO_NAMES[info[0]], "cluster": info[1], "w_ring": info[2], "batch_slices": info[3],
                "small_kernel": bool(info[4]), "w_hh_resident": info[0] == 2 and info[2] == 0,
                "layer_wave": bool(info[5]), "wave_ctas_per_sm": int(info[6])}

    def last_launch_count(self) -> int:
        """Kernels the library launched in the last forward call on this
        thread (``hs_rnn_last_launch_count``; memsets and copies excluded)."""
        return int(self.lib.hs_rnn_last_launch_count())

    def alloc_outputs(self, batch: int | None = None):
        s = self.spec
        B = s.batch if batch is None else batch
        y = torch.empty((s.seq, B, s.dirs * s.hidden), device=self.device)
        hn = torch.empty((s.layers * s.dirs, B, s.hidden), device=self.device)
        cn = torch.empty_like(hn) if s.cell == "lstm" else None
        return y, hn, cn

    def _check_dev(self, name, t, shape, required=False):
        """Every tensor handed to the library as a raw pointer: float32,
        contiguous, on this executor's device, of the expected shape."""
        if t is None:
            if required:
                raise ValueError(f"{name} is required")
            return
        if t.device != self.device or t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous float32 tensor on {self.device} "
                             f"(got {t.dtype} on {t.device}, contiguous={t.is_contiguous()})")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")

    def forward(self, x: torch.Tensor, h0=None, c0=None, out=None, layer_ms: bool = False):
        """Run the DAG on device tensors.  Returns ``(y, h_n, c_n)`` (c_n None
        for GRU), plus per-layer [gemm_ms, recurrent_ms] when ``layer_ms``."""
        self._require_resident()
        s = self.spec
        if x.device != self.device or x.dtype != torch.float32 or not x.is_contiguous():
            raise ValueError("x must be a contiguous float32 tensor on the executor's device")
        if tuple(x.shape) != (s.seq, s.batch, s.I):
            raise ValueError(f"x has shape {tuple(x.shape)}, expected {(s.seq, s.batch, s.I)}")
        state = (s.layers * s.dirs, s.batch, s.hidden)
        self._check_dev("h0", h0, state)
        self._check_dev("c0", c0 if s.cell == "lstm" else None, state)
        y, hn, cn = out if out is not None else self.alloc_outputs()
        self._check_dev("y", y, (s.seq, s.batch, s.dirs * s.hidden), required=True)
        self._check_dev("h_n", hn, state, required=True)
        self._check_dev("c_n", cn, state, required=s.cell == "lstm")
        times = (ctypes.c_float * (2 * s.layers))() if layer_ms else None
        ptr = lambda t: t.data_ptr() if t is not None else None
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            _check(
                self.lib,
                "hs_rnn_forward_packed",
                self.lib.hs_rnn_forward_packed(
                    ctypes.byref(self.desc), self.packed.data_ptr(), x.data_ptr(), ptr(h0), ptr(c0),
                    y.data_ptr(), hn.data_ptr(), ptr(cn), self.workspace.data_ptr(), self.workspace.numel(),
                    stream.cuda_stream, times,
                ),
            )
        if layer_ms:
            return y, hn, cn, [[times[2 * l], times[2 * l + 1]] for l in range(s.layers)]
        return y, hn, cn

    def graph(self, h0=None, c0=None, warmup: int = 2) -> "GraphedForward":
        """Capture one device forward into a CUDA graph (``torch.cuda.CUDAGraph``).

        Launch-bound shapes (small layers, short sequences: the per-request
        models of a serving loop) pay their launch and host costs once at
        capture; ``GraphedForward.replay`` then re-runs every kernel of the
        forward with one graph launch.  The captured forward runs its layers
        back to back on one stream: the overlapped schedules (next-layer K1 and
        XP streaming on a second stream, which spin on each other's progress
        counters) are off, since a graph may start sibling nodes in either
        order.  The results are bit-identical to ``forward`` (same tiles, same
        accumulation order).  ``h0`` / ``c0`` are captured by address."""
        self._require_resident()
        s = self.spec
        state = (s.layers * s.dirs, s.batch, s.hidden)
        self._check_dev("h0", h0, state)
        self._check_dev("c0", c0 if s.cell == "lstm" else None, state)
        x = torch.zeros((s.seq, s.batch, s.I), device=self.device)
        out = self.alloc_outputs()
        with torch.cuda.device(self.device):
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):  # plans, lazy module loads, one-time probes: before the capture
                for _ in range(max(1, warmup)):
                    self.forward(x, h0, c0, out=out)
            torch.cuda.current_stream(self.device).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.forward(x, h0, c0, out=out)
        return GraphedForward(g, x, out)

    def profile_cells(self, x: torch.Tensor, h0=None, c0=None, out=None):
        """Per-cell GPU cost (ms) of the whole-DAG forward, ``hs_rnn_profile_cells``:
        ``[layers*dirs*T]`` indexed like the cell grid's nodes, summing to the
        measured forward.  Returns ``(cell_ms, forward_ms)``."""
        self._require_resident()
        s = self.spec
        if x.device != self.device or x.dtype != torch.float32 or not x.is_contiguous():
            raise ValueError("x must be a contiguous float32 tensor on the executor's device")
        if tuple(x.shape) != (s.seq, s.batch, s.I):
            raise ValueError(f"x has shape {tuple(x.shape)}, expected {(s.seq, s.batch, s.I)}")
        state = (s.layers * s.dirs, s.batch, s.hidden)
        self._check_dev("h0", h0, state)
        self._check_dev("c0", c0 if s.cell == "lstm" else None, state)
        y, hn, cn = out if out is not None else self.alloc_outputs()
        n = s.layers * s.dirs * s.seq
        cells = (ctypes.c_float * n)()
        fwd = ctypes.c_float()
        ptr = lambda t: t.data_ptr() if t is not None else None
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            _check(
                self.lib,
                "hs_rnn_profile_cells",
                self.lib.hs_rnn_profile_cells(
                    ctypes.byref(self.desc), self.packed.data_ptr(), x.data_ptr(), ptr(h0), ptr(c0),
                    y.data_ptr(), hn.data_ptr(), ptr(cn), self.workspace.data_ptr(), self.workspace.numel(),
                    stream.cuda_stream, cells, ctypes.byref(fwd),
                ),
            )
        return [float(v) for v in cells], float(fwd.value)

    def alloc_host_outputs(self):
        """Pinned host output buffers (y, h_n, c_n) for :meth:`forward_host`."""
        return tuple(torch.empty(t.shape, dtype=t.dtype).pin_memory() if t is not None else None
                     for t in self.alloc_outputs())

    def outputs_ready(self, y_host: torch.Tensor, stream=None):
        """Wait for the output copies of an ``async_outputs`` :meth:`forward_host`
        into ``y_host``: make ``stream`` wait (GPU side), or block the calling
        thread when ``stream`` is None (``hs_rnn_outputs_ready``)."""
        _check(self.lib, "hs_rnn_outputs_ready",
               self.lib.hs_rnn_outputs_ready(y_host.data_ptr(), stream.cuda_stream if stream is not None else None))

    def forward_host(self, x_host: torch.Tensor, h0=None, c0=None, out_host=None, staging=None, upload_chunks=0,
                     async_outputs=False):
        """End-to-end forward on host tensors (``hs_rnn_forward_host``): the
        H2D upload of ``x`` and the D2H download of ``y`` overlap the compute
        on the tensor-core path.  Host tensors should be pinned.  Returns the
        host ``(y, h_n, c_n)``; work is complete when the current stream is.
        ``upload_chunks``: time chunks x is uploaded in (0 = library default);
        1 suits request streams, where the upload overlaps the previous request."""
        self._require_resident()
        s = self.spec
        for name, t in (("x", x_host), ("h0", h0), ("c0", c0)):
            if t is not None and (t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous float32 host tensor")
        if tuple(x_host.shape) != (s.seq, s.batch, s.I):
            raise ValueError(f"x has shape {tuple(x_host.shape)}, expected {(s.seq, s.batch, s.I)}")
        y, hn, cn = out_host if out_host is not None else self.alloc_host_outputs()
        state = (s.layers * s.dirs, s.batch, s.hidden)
        for name, t, shp, req in (("y", y, (s.seq, s.batch, s.dirs * s.hidden), True), ("h_n", hn, state, True),
                                  ("c_n", cn, state, s.cell == "lstm"), ("h0", h0, state, False),
                                  ("c0", c0, state, False)):
            if t is None:
                if req:
                    raise ValueError(f"{name} is required")
                continue
            if t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous() or tuple(t.shape) != shp:
                raise ValueError(f"{name} must be a contiguous float32 host tensor of shape {shp}")
        if staging is None:
            staging = self.alloc_staging()
        xd, (yd, hnd, cnd), state = staging
        ptr = lambda t: t.data_ptr() if t is not None else None
        desc = make_desc(s)  # per call: concurrent callers never share a mutated descriptor
        desc.upload_chunks = int(upload_chunks)
        desc.async_outputs = 1 if async_outputs else 0
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            _check(
                self.lib,
                "hs_rnn_forward_host",
                self.lib.hs_rnn_forward_host(
                    ctypes.byref(desc), self.packed.data_ptr(), x_host.data_ptr(), ptr(h0), ptr(c0),
                    y.data_ptr(), hn.data_ptr(), ptr(cn), xd.data_ptr(), yd.data_ptr(), hnd.data_ptr(), ptr(cnd),
                    state.data_ptr(), self.workspace.data_ptr(), self.workspace.numel(), stream.cuda_stream,
                ),
            )
        return y, hn, cn

    def forward_stage(self, link: "StageLink", x=None, h0=None, c0=None, out=None):
        """One layer-pipeline stage (``hs_rnn_forward_stage``): input from
        ``link.x_planes`` (or ``x``), output shipped to the next stage through
        ``link``; returns ``(y, h_n, c_n)`` of this stage's layers."""
        self._require_resident()
        s = self.spec
        if x is not None:
            if x.device != self.device or x.dtype != torch.float32 or not x.is_contiguous():
                raise ValueError("x must be a contiguous float32 tensor on the executor's device")
            if tuple(x.shape) != (s.seq, s.batch, s.I):
                raise ValueError(f"x has shape {tuple(x.shape)}, expected {(s.seq, s.batch, s.I)}")
        elif not link.x_planes:
            raise ValueError("a stage needs x or link.x_planes")
        state = (s.layers * s.dirs, s.batch, s.hidden)
        self._check_dev("h0", h0, state)
        self._check_dev("c0", c0 if s.cell == "lstm" else None, state)
        y, hn, cn = out if out is not None else self.alloc_outputs()
        ptr = lambda t: t.data_ptr() if t is not None else None
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            _check(
                self.lib,
                "hs_rnn_forward_stage",
                self.lib.hs_rnn_forward_stage(
                    ctypes.byref(self.desc), self.packed.data_ptr(), ptr(x), ptr(h0), ptr(c0),
                    y.data_ptr(), hn.data_ptr(), ptr(cn), ctypes.byref(link), self.workspace.data_ptr(),
                    self.workspace.numel(), stream.cuda_stream,
                ),
            )
        return y, hn, cn

    def alloc_staging(self):
        """Device staging buffers for :meth:`forward_host`: (x, (y, h_n, c_n), states)."""
        s = self.spec
        xd = torch.empty((s.seq, s.batch, s.I), device=self.device)
        state = torch.empty((2, s.layers * s.dirs, s.batch, s.hidden), device=self.device)
        return xd, self.alloc_outputs(), state

    def run_cells(self, ld: int, t0: int, t1: int, inp, out, h_prev, c_prev, h_last, c_last, stream=None):
        """Steps ``t0..t1-1`` (processing order) of layer-direction ``ld``, on
        ``stream`` (a ``torch.cuda.Stream`` of this executor's device; default:
        the device's current stream).  The hybrid executor passes its stream so
        a segment's dispatch skips the device-context switch."""
        self._require_resident()
        ptr = lambda t: t.data_ptr() if t is not None else None
        if stream is None:
            with torch.cuda.device(self.device):
                stream = torch.cuda.current_stream(self.device)
        elif (self.device.index is not None and
              (stream.device.index != self.device.index or torch.cuda.current_device() != self.device.index)):
            raise ValueError(f"run_cells(stream=...) needs a stream of {self.device} and that device current "
                             f"(got a stream on {stream.device}, current device {torch.cuda.current_device()})")
        _check(
            self.lib,
            "hs_rnn_run_cells",
            self.lib.hs_rnn_run_cells(
                ctypes.byref(self.desc), self.packed.data_ptr(), ld, t0, t1, ptr(inp), ptr(out),
                ptr(h_prev), ptr(c_prev), ptr(h_last), ptr(c_last), self.workspace.data_ptr(),
                self.workspace.numel(), stream.cuda_stream,
            ),
        )
