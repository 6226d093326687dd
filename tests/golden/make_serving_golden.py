"""Generate tests/golden/serving_golden.json by running the REFERENCE CLI.

Run in the build container only (needs /root/reference):
    python tests/golden/make_serving_golden.py

Each corpus scenario is written as a scenario file and served by the
unmodified reference's own command (`hetsched serve --scenario ... --no-figure`,
cli.py:383-445 -> servingsim.run_serving / compare_patterns,
servingsim.py:143-288).  The metrics.json and every events CSV are recorded
byte for byte; tests/test_serving_golden.py loads the same scenario files with
this package and requires identical text.
"""
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).with_name("serving_golden.json")


def _models(n, foot, exec_ms, weights, slo_mult, seed):
    import numpy as np

    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        f = float(round(foot * (0.5 + rng.random()), 3))
        e = float(round(exec_ms * (0.5 + rng.random()), 4))
        w = float(round(weights * (0.5 + rng.random()), 3))
        out.append({"id": f"m{i}", "gpu_footprint_mb": f, "exec_latency_ms": e, "weights_mb": w,
                    "slo_ms": float(round(e * slo_mult * (1.0 + 5.0 * rng.random()), 4))})
    return out


def corpus():
    cases = []
    for i, (n, cap, pat, seed, ia, foot) in enumerate([
        (3, 1000.0, "uniform", 0, 0.0, 400.0),
        (4, 1000.0, "random", 4, 0.0, 350.0),
        (9, 2000.0, "uniform", 0, 0.0, 500.0),      # the paper's nine-model uniform study
        (9, 2000.0, "random", 11, 2.5, 500.0),
        (5, 700.0, "random", 3, 7.0, 300.0),
        (2, 1000.0, "uniform", 0, 4.0, 600.0),
    ]):
        models = _models(n, foot, 10.0, foot * 0.6, 1.25, 100 + i)
        cases.append({"capacity_mb": cap, "bandwidth_mb_per_ms": 12.0 + i,
                      "workload": {"total_requests": 60 + 7 * i, "pattern": pat, "seed": seed, "interarrival_ms": ia},
                      "models": models})
    # pattern comparisons (Table 6 shape): the latency-optimal variant is faster
    # and smaller, the memory-optimal variant smaller still but slower
    for i, (n, cap, pat, seed) in enumerate([(9, 2500.0, "uniform", 0), (6, 1500.0, "random", 5)]):
        g = _models(n, 500.0, 10.0, 300.0, 1.25, 200 + i)
        lat = [dict(m, gpu_footprint_mb=m["gpu_footprint_mb"] * 0.7, exec_latency_ms=m["exec_latency_ms"] * 0.85,
                    weights_mb=m["weights_mb"] * 0.7) for m in g]
        mem = [dict(m, gpu_footprint_mb=m["gpu_footprint_mb"] * 0.4, exec_latency_ms=m["exec_latency_ms"] * 1.15,
                    weights_mb=m["weights_mb"] * 0.4) for m in g]
        cases.append({"capacity_mb": cap, "bandwidth_mb_per_ms": 12.0,
                      "workload": {"total_requests": 90, "pattern": pat, "seed": seed, "interarrival_ms": 0.0},
                      "patterns": {"gpu": g, "latency-optimal": lat, "memory-optimal": mem}})
    return cases


def main():
    sys.path.insert(0, str(REF))
    import hetsched

    out = {"generator": "tests/golden/make_serving_golden.py", "reference": "hetsched " + hetsched.__version__,
           "cases": []}
    env = dict(os.environ, PYTHONPATH=str(REF))
    for sc in corpus():
        with tempfile.TemporaryDirectory() as d:
            f = Path(d) / "scenario.json"
            f.write_text(json.dumps(sc))
            od = Path(d) / "out"
            r = subprocess.run([sys.executable, "-m", "hetsched.cli", "serve", "--scenario", str(f), "--no-figure",
                                "--out", str(od)], cwd=d, env=env, capture_output=True, text=True)
            if r.returncode:
                raise RuntimeError(r.stderr)
            files = {p.name: p.read_text() for p in sorted(od.iterdir()) if p.suffix in (".csv", ".json")
                     and not p.name.endswith("config.json")}
            out["cases"].append({"scenario": sc, "stdout": r.stdout, "files": files})
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {OUT} ({len(out['cases'])} cases)")


if __name__ == "__main__":
    main()
