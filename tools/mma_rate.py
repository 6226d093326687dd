"""tcgen05.mma rate at the recurrence's shapes (tools/probe/mma_rate.cu):
cycles per M=128, K=16 kind::f16 MMA issued back to back by one thread, A
from shared memory (SS) or tensor memory (TS), N = 16..256, 1/2/4 accumulators;
and in chunks of 8 with the recurrence loop's per-chunk barrier waits / commits,
alone or with 8 more warps of the CTA waiting on an mbarrier meanwhile.

usage: python tools/mma_rate.py [out.json]   (builds the probe with nvcc)"""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tools" / "probe" / "mma_rate.cu"
LIB = ROOT / "tools" / "probe" / "libmmarate.so"


def build():
    if LIB.exists() and LIB.stat().st_mtime > SRC.stat().st_mtime:
        return
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                    "-Xcompiler", "-fPIC", "-o", str(LIB), str(SRC)], check=True)


def main():
    build()
    if len(sys.argv) > 1 and sys.argv[1] == "--build":
        return
    lib = ctypes.CDLL(str(LIB))
    d = ctypes.c_double
    lib.mma_rate.argtypes = [ctypes.c_int] * 6 + [ctypes.POINTER(d)] * 2
    rows = []
    for ts in (0, 1, 2, 3, 4, 5, 6, 7):
        for N in ((16, 32, 64, 128, 256) if ts < 2 else (16, 32)):
            for nacc in ((1, 2, 4) if ts < 4 else (1,)):
                if nacc * N > 256:
                    continue
                for grid, threads in ((148, 128), (148, 288)):
                    if threads > 128 and ts < 4:
                        continue
                    a, b = d(), d()
                    rc = lib.mma_rate(ts, N, 4096, nacc, grid, threads, ctypes.byref(a), ctypes.byref(b))
                    assert rc == 0, rc
                    r = {"threads": threads, "mode": ["SS", "TS", "TS chunks of 8 (1 wait)", "SS chunks of 8 (2 waits + commit)",
                                             "TS unrolled chunks", "TS unrolled chunks + wait",
                                             "SS unrolled chunks", "SS unrolled chunks + 2 waits + commit"][ts], "N": N, "nacc": nacc, "ctas": grid,
                         "issue_cyc_per_mma": round(a.value, 2), "cyc_per_mma": round(b.value, 2),
                         "floor_cyc": 128 * N / 256}
                    rows.append(r)
                    print(json.dumps(r), flush=True)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
