"""Generate tests/golden/sweep_golden.json by running the REFERENCE CLI.

Run in the build container only (needs /root/reference):
    python tests/golden/make_sweep_golden.py

For each corpus entry it runs the unmodified reference's own commands
(`hetsched gen-graph`, `gen-profile`, `sweep --no-figure`, cli.py:259-306 with
the `_alpha_range` grid of cli.py:125-140) in a scratch directory and records
the sweep.csv text byte for byte.  tests/test_sweep_golden.py rebuilds the
same graph/profile with this package and requires planner.sweep_csv to
produce identical text.
"""
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).with_name("sweep_golden.json")

# (graph args, profile preset, profile seed, alpha spec, io_transfers)
CORPUS = [
    (["--family", "lstm", "--layers", "1", "--seq", "16"], "cpu-comparable", 0, "0:1:0.1", False),   # c1 grid
    (["--family", "lstm", "--layers", "1", "--seq", "16"], "gpu-dominant", 3, "0:1:0.1", True),
    (["--family", "lstm", "--layers", "2", "--seq", "128"], "cpu-comparable", 0, "0:1:0.1", False),  # c2 grid
    (["--family", "lstm", "--layers", "2", "--seq", "128"], "comm-heavy", 1, "0:2:0.25", True),
    (["--family", "lstm", "--layers", "4", "--seq", "256"], "cpu-comparable", 0, "0:1:0.1", False),  # c3 grid
    (["--family", "lstm", "--layers", "4", "--seq", "64"], "cpu-comparable", 7, "0:5:0.5", False),
    (["--family", "demo7"], "cpu-comparable", 0, "0:1:0.1", False),
    (["--family", "demo7"], "comm-heavy", 5, "0:3:0.3", True),
    (["--family", "random", "--nodes", "30", "--edge-prob", "0.2", "--seed", "4"], "cpu-comparable", 2, "0:1:0.1", False),
    (["--family", "random", "--nodes", "12", "--edge-prob", "0.4", "--seed", "9"], "gpu-dominant", 8, "0.5:1.5:0.125", True),
]


def run(args, cwd):
    env = dict(os.environ, PYTHONPATH=str(REF))
    r = subprocess.run([sys.executable, "-m", "hetsched.cli", *args], cwd=cwd, env=env, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"{args}: {r.stderr}")
    return r.stdout


def main():
    sys.path.insert(0, str(REF))
    import hetsched

    out = {"generator": "tests/golden/make_sweep_golden.py", "reference": "hetsched " + hetsched.__version__, "cases": []}
    for gargs, preset, pseed, alphas, io in CORPUS:
        with tempfile.TemporaryDirectory() as d:
            run(["gen-graph", *gargs, "--out", d], d)
            gfile = Path(d) / "graph.json"
            run(["gen-profile", "--graph", str(gfile), "--preset", preset, "--seed", str(pseed), "--out", d], d)
            pfile = Path(d) / "profile.json"
            sd = Path(d) / "sweep"
            sd.mkdir()
            run(["sweep", "--graph", str(gfile), "--profile", str(pfile), "--alpha-sweep", alphas, "--no-figure",
                 "--out", str(sd)] + (["--io-transfers"] if io else []), d)
            out["cases"].append({"graph_args": gargs, "preset": preset, "profile_seed": pseed,
                                 "alphas": alphas, "io_transfers": io, "sweep_csv": (sd / "sweep.csv").read_text()})
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {OUT} ({len(out['cases'])} cases)")


if __name__ == "__main__":
    main()
