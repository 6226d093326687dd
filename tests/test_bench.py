"""bench.py's roofline arithmetic (pure host code, no GPU)."""
import importlib.util
from pathlib import Path

import pytest

from paper_2307_11339_b200 import CONFIGS

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_roofline_entry_c2_resident():
    b = _bench()
    spec = CONFIGS["c2"]
    peaks = {"bf16_tflops": 1618.9, "hbm_gbs": 6548.5, "source": "measured"}
    rec_f = 2.0 * spec.G * spec.hidden * spec.hidden * spec.batch * spec.seq * spec.layers
    r = b.roofline_entry(spec, {"w_ring": 0, "batch_slices": 1}, "tc", rec_f, 1.5, 0.15, peaks, None, sm_mhz=1965.0, sms=148)
    assert r["bound"] == "tensor"
    assert r["frac"] == pytest.approx(rec_f / 1.5e-3 / 1e12 / 1618.9)
    sv = r["survey_fp32_roofline"]
    p_ffma = 148 * 128 * 2 * 1965e6
    assert sv["p_ffma_tflops"] == pytest.approx(p_ffma / 1e12)
    assert sv["t_roof_ms"] == pytest.approx(rec_f / p_ffma * 1e3)  # W_hh resident: no byte term
    assert sv["frac"] == pytest.approx(rec_f / p_ffma / 1.5e-3)


def test_roofline_entry_streamed_w_is_l2_traffic():
    """c4: the W_hh ring re-reads hit L2 (ncu r02), so the HBM leg counts W
    once per launch and the per-step re-reads go to the "l2" leg."""
    b = _bench()
    spec = CONFIGS["c4"]
    peaks = {"bf16_tflops": 1618.9, "hbm_gbs": 6548.5, "source": "measured"}
    rec_f = 2.0 * spec.G * spec.hidden * spec.hidden * spec.batch * spec.seq * spec.layers
    l2 = {"gbs": 24400.0, "source": "ncu"}
    r = b.roofline_entry(spec, {"w_ring": 4, "batch_slices": 1}, "tc", rec_f, 32.0, 1.3, peaks, None, sm_mhz=1965.0,
                         l2_peak=l2)
    wbytes = 4.0 * 4 * 2048 * 2048
    hbm = spec.seq * 8 * (4.0 * 16 * 4 * 2048 + 4.0 * 16 * 2048) + wbytes * 8
    other = r if r["bound"] == "hbm" else r["other"]
    assert other["algorithmic_bytes"] == pytest.approx(hbm)
    assert r["l2"]["bytes"] == pytest.approx(wbytes * spec.seq * 8)
    assert r["l2"]["frac"] == pytest.approx(wbytes * spec.seq * 8 / 32e-3 / 1e9 / 24400.0)
    assert r["survey_fp32_roofline"]["t_roof_ms"] > 40.0  # the SURVEY formula still charges HBM per step
