"""Debug: per-step precision of the tensor-core recurrence vs CPU emulations."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.rnn_ref import rnn_forward_ref  # noqa: E402
from paper_2307_11339_b200 import RNNExecutor, RNNSpec, init_weights, make_input  # noqa: E402

for T in (1, 2, 8, 32):
    spec = RNNSpec("lstm", 1, 1024, T, 64, algo="tc")
    w = init_weights(spec, 0)
    x = make_input(spec, 1)
    ex = RNNExecutor(spec, w)
    y = ex.forward(x.cuda())[0].cpu().double()
    ry = rnn_forward_ref("lstm", x.double().numpy(), [{k: v.double().numpy() for k, v in d.items()} for d in w])[0]

    def emu(hq, wq):
        W = w[0]
        Whh = wq(W["w_hh"].double())
        xp = x.double() @ W["w_ih"].double().T + W["b_ih"].double() + W["b_hh"].double()
        H = 1024
        h = torch.zeros(64, H, dtype=torch.float64)
        c = torch.zeros_like(h)
        out = []
        for t in range(T):
            g = xp[t] + hq(h) @ Whh.T
            i, f, gg, o = g.split(H, 1)
            c = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(gg)
            h = torch.sigmoid(o) * torch.tanh(c)
            out.append(h)
        return torch.stack(out).numpy()

    s16 = lambda t: t.half().double() + (t - t.half().double()).half().double()
    e_full = emu(lambda h: h.half().double(), s16)
    e_hi = emu(lambda h: h.half().double(), lambda t: t.half().double())
    print(f"T={T}: gpu-oracle {np.abs(y.numpy() - ry).max():.2e}  emu(hi+lo)-oracle {np.abs(e_full - ry).max():.2e}  "
          f"emu(hi only)-oracle {np.abs(e_hi - ry).max():.2e}  gpu-emu(hi+lo) {np.abs(y.numpy() - e_full).max():.2e}  "
          f"gpu-emu(hi) {np.abs(y.numpy() - e_hi).max():.2e}")
