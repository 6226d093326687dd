"""Measure the peaks MEASURED_PEAKS.json lacks: FP32 FFMA
TFLOP/s and the L2 read bandwidth of an L2-resident working set (64 MiB, the
c4 W_hh planes), beside an HBM-sized read (4 GiB).  Writes
profiles/peaks_fp32_l2.json, which bench.py's rooflines read.

usage: python tools/peak_probe.py [out.json]   (builds tools/probe/peaks.cu with nvcc)"""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tools" / "probe" / "peaks.cu"
LIB = ROOT / "tools" / "probe" / "libpeaks.so"


def main():
    if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                               "-fPIC", "-o", str(LIB), str(SRC)])
    lib = ctypes.CDLL(str(LIB))
    lib.probe_ffma_tflops.restype = ctypes.c_float
    lib.probe_read_gbs.restype = ctypes.c_float
    lib.probe_read_gbs.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
    import torch

    clocks = None
    try:
        import pynvml as nv

        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
        clocks = {"sm_mhz_after": nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                  "sm_max_mhz": nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)}
    except Exception:
        pass
    out = {
        "gpu": torch.cuda.get_device_name(0),
        "ffma_tflops": float(lib.probe_ffma_tflops(5)),
        "l2_read_gbs_64MiB": float(lib.probe_read_gbs(64 << 20, 20, 5)),
        "hbm_read_gbs_4GiB": float(lib.probe_read_gbs(4 << 30, 1, 5)),
        "clocks": clocks,
        "how": "tools/probe/peaks.cu: 8 independent FFMA chains x 2^14 iterations on 8 CTAs x 256 threads per SM; "
               "ld.global.cg 16-B vector reads over a buffer re-read 20x (64 MiB, L2-resident) or once (4 GiB); "
               "best of 5, CUDA events",
    }
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
