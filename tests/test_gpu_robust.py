"""Forward progress of the persistent kernels.

The recurrences are persistent grids whose CTAs wait on each other through
global counters; they launch cooperatively (all CTAs resident or none) and
every cross-CTA / cross-kernel spin is bounded by the watchdog in common.cuh.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.rnn_ref import rnn_forward_ref
from paper_2307_11339_b200 import CONFIGS, RNNExecutor, RNNSpec, init_weights, make_input

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_watchdog_turns_a_stall_into_an_error():
    """A recurrence waiting for K1 tiles that never arrive (HS_TEST_STALL)
    must end in a CUDA error whose message names the watchdog site, not hang."""
    code = (
        "import sys, torch; sys.path.insert(0, '.');"
        "from paper_2307_11339_b200 import RNNExecutor, RNNSpec, init_weights, make_input;"
        "from paper_2307_11339_b200.rnn import HsRnnError;"
        "s = RNNSpec('lstm', 1, 256, 8, 16, algo='tc');"
        "ex = RNNExecutor(s, init_weights(s, 0)); x = make_input(s, 1).cuda();\n"
        "try:\n"
        "    ex.forward(x); torch.cuda.synchronize(); print('NO-ERROR')\n"
        "except Exception as e:\n"
        "    print('SYNC-ERROR', type(e).__name__)\n"
        "try:\n"
        "    ex.forward(x); print('NO-ERROR-2')\n"
        "except HsRnnError as e:\n"
        "    print('LIB-ERROR', e)\n"
    )
    env = dict(os.environ, HS_TEST_STALL="1", HS_WATCHDOG_MS="300")
    p = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=300)
    print(p.stdout, p.stderr[-2000:])
    assert "SYNC-ERROR" in p.stdout
    assert "LIB-ERROR" in p.stdout and "watchdog" in p.stdout and "XP readiness" in p.stdout


def test_forward_beside_a_competing_kernel():
    """A forward enqueued while another stream keeps the SMs busy with GEMMs
    either completes correctly (the cooperative launch waits for room) or
    errors cleanly; it never hangs (subprocess with a deadline)."""
    code = (
        "import sys, torch, numpy as np; sys.path.insert(0, '.');"
        "from paper_2307_11339_b200 import RNNExecutor, CONFIGS, init_weights, make_input;"
        "s = CONFIGS['c2'].with_(seq=32);"
        "ex = RNNExecutor(s, init_weights(s, 0)); x = make_input(s, 1).cuda();"
        "ref = [t.clone() for t in ex.forward(x)]; torch.cuda.synchronize();"
        "other = torch.cuda.Stream(); a = torch.randn(8192, 8192, device='cuda');"
        "ok = 0\n"
        "for i in range(5):\n"
        "    with torch.cuda.stream(other):\n"
        "        for _ in range(8): b = a @ a\n"
        "    got = ex.forward(x); torch.cuda.synchronize()\n"
        "    ok += all(torch.equal(g, r) for g, r in zip(got, ref))\n"
        "print('OK', ok)\n"
    )
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(p.stdout, p.stderr[-2000:])
    assert "OK 5" in p.stdout


def test_persistent_launch_is_cooperative_and_correct():
    """The cooperative + cluster launch of both recurrence forms (single-group
    c3 shape, two-group c2 shape) at reduced T matches the oracle."""
    for spec in (CONFIGS["c3"].with_(seq=16), CONFIGS["c2"].with_(seq=16)):
        w = init_weights(spec, 0)
        x = make_input(spec, 1)
        ex = RNNExecutor(spec, w)
        y, hn, cn = ex.forward(x.to(ex.device))
        ry, rh, rc = rnn_forward_ref(spec.cell, x.double().numpy(),
                                     [{k: v.double().numpy() for k, v in d.items()} for d in w])
        assert float(np.abs(y.cpu().double().numpy() - ry).max()) <= 1e-4
        assert float(np.abs(hn.cpu().double().numpy() - rh).max()) <= 1e-4
