"""C-ABI boundary checks that need no GPU: the in-tree library loads, exports
every symbol include/hs_rnn.h declares, and validates descriptors."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2307_11339_b200 import CONFIGS, RNNSpec, load_library, rnn

HEADER = Path(__file__).resolve().parents[1] / "include" / "hs_rnn.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(hs_\w+)\s*\(", text, re.M)))


def test_header_symbols_match_binding_list():
    assert declared_symbols() == sorted(rnn.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.hs_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess, shutil
    lib = Path(rnn._build.library_path())
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", str(lib)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def _ws(spec):
    lib = load_library()
    d = rnn.make_desc(spec)
    n = ctypes.c_size_t()
    rc = lib.hs_rnn_workspace(ctypes.byref(d), ctypes.byref(n))
    return rc, n.value, lib.hs_last_error().decode()


def test_workspace_sizes_scale_with_config():
    rc, ws2, _ = _ws(CONFIGS["c2"])
    assert rc == 0
    # xproj dominates: T*B*4H floats = 128*64*4096*4 bytes = 128 MiB
    assert ws2 >= 128 * 64 * 4096 * 4
    rc, ws1, _ = _ws(CONFIGS["c1"])
    assert rc == 0 and ws1 < ws2


@pytest.mark.parametrize(
    "field,value,code",
    [("cell", 7, 1), ("layers", 0, 1), ("dirs", 3, 1), ("batch", 0, 1), ("dtype", 9, 1), ("algo", 5, 1), ("hidden", 30, 3)],
)
def test_descriptor_validation(field, value, code):
    lib = load_library()
    d = rnn.make_desc(CONFIGS["c1"])
    setattr(d, field, value)
    n = ctypes.c_size_t()
    assert lib.hs_rnn_workspace(ctypes.byref(d), ctypes.byref(n)) == code
    assert lib.hs_last_error()


def test_null_descriptor_rejected():
    lib = load_library()
    n = ctypes.c_size_t()
    assert lib.hs_rnn_workspace(None, ctypes.byref(n)) == 1
    assert b"NULL" in lib.hs_last_error()


def test_forward_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        rnn.RNNExecutor(CONFIGS["c1"], rnn.init_weights(CONFIGS["c1"]))


def test_plan_query_without_gpu():
    """hs_rnn_plan is static (no device needed): the BASELINE configs map to
    the kernels DESIGN.md describes."""
    import ctypes

    from paper_2307_11339_b200 import CONFIGS
    from paper_2307_11339_b200.rnn import load_library, make_desc

    lib = load_library()

    def plan(spec):
        info = (ctypes.c_int32 * 8)()
        assert lib.hs_rnn_plan(ctypes.byref(make_desc(spec)), info) == 0
        return list(info)

    c1, c2, c3, c4, c5 = (plan(CONFIGS[k]) for k in ("c1", "c2", "c3", "c4", "c5"))
    assert c1[0] == 1 and c1[4] == 1 and c1[1] in (4, 8, 16)  # SIMT small-shape cluster kernel
    assert c2[0] == 2 and c2[2] == 0 and c2[1] == 4          # tensor cores, W_hh resident, S = 4
    assert c3[0] == 2 and c3[2] == 0
    assert c4[0] == 2 and c4[2] > 0                          # W_hh 64 MiB/layer: streamed ring
    assert c5[0] == 2 and c5[3] > 1                          # bf16, batch sliced on one GPU


def test_integration_stub_descriptor_matches_the_header():
    """The ctypes stub INTEGRATION.md shows a maintainer declares the same
    descriptor layout as include/hs_rnn.h (and the package's own binding)."""
    doc = (HEADER.parents[1] / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n(import ctypes\n\nclass hs_rnn_desc.*?)\nlib = ", doc, re.S).group(1)
    ns = {}
    exec(block, ns)
    stub = ns["hs_rnn_desc"]
    assert ctypes.sizeof(stub) == ctypes.sizeof(rnn._Desc)
    hdr = HEADER.read_text()
    body = re.search(r"typedef struct hs_rnn_desc \{(.*?)\} hs_rnn_desc;", hdr, re.S).group(1)
    named = re.findall(r"int32_t (\w+);", body)
    assert [f[0] for f in stub._fields_ if f[0] != "reserved"] == named
    assert [f[0] for f in rnn._Desc._fields_ if f[0] != "reserved"] == named
