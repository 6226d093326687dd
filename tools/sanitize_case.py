"""Small forwards through every kernel family, for compute-sanitizer runs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_11339_b200 import RNNExecutor, RNNSpec, init_weights, make_input  # noqa: E402

for spec in (RNNSpec("lstm", 2, 256, 4, 16, algo="tc"), RNNSpec("gru", 2, 128, 3, 8, dirs=2, algo="tc"),
             RNNSpec("lstm", 2, 64, 4, 4, algo="simt")):
    ex = RNNExecutor(spec, init_weights(spec))
    x = make_input(spec)
    ex.forward(x.cuda())
    ex.forward_host(x.pin_memory())
    torch.cuda.synchronize()
    print("ok", spec)
