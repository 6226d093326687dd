"""CPU emulation (float64 with fp16 operand rounding) of the f32-mode operand
schemes: per-layer h_n / c_n max-abs against the exact recurrence for the K1
input rounded to fp16 in every layer, or in layers >= 1 only (the dropped
two-pass K1 experiment, profiles/r02_k1_fp16_twopass.txt).

  python tools/k1_precision_emu.py L H T B      (c2: 2 1024 128 64)
"""
import sys
import time

import numpy as np
import torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_11339_b200 import RNNSpec, init_weights, make_input
torch.set_num_threads(16)
L, H, T, B = [int(v) for v in sys.argv[1:5]]
spec = RNNSpec("lstm", L, H, T, B)
w = init_weights(spec, 0)
x = make_input(spec, 1).double()
def s16(t):
    hi = t.half().double(); return hi + (t - hi).half().double()
def run(xq_of_layer, exact=False):
    inp = x; hns=[]; cns=[]
    for l in range(L):
        W = w[l]
        Wih = W["w_ih"].double() if exact else s16(W["w_ih"].double())
        Whh = W["w_hh"].double() if exact else s16(W["w_hh"].double())
        xp = xq_of_layer(l)(inp) @ Wih.T + W["b_ih"].double() + W["b_hh"].double()
        h = torch.zeros(B, H, dtype=torch.float64); c = torch.zeros_like(h); out = []
        for t in range(T):
            g = xp[t] + (h if exact else h.half().double()) @ Whh.T
            i, f, gg, o = g.split(H, 1)
            c = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(gg)
            h = torch.sigmoid(o) * torch.tanh(c); out.append(h)
        inp = torch.stack(out); hns.append(h); cns.append(c)
    return inp.numpy(), [v.numpy() for v in hns], [v.numpy() for v in cns]
ident = lambda v: v
f16 = lambda v: v.half().double()
o = run(lambda l: ident, exact=True)
def rep(name, r):
    print(f"{name}: y {np.abs(r[0]-o[0]).max():.2e} hn " + " ".join(f"{np.abs(a-b).max():.1e}" for a,b in zip(r[1],o[1])) +
          " | cn " + " ".join(f"{np.abs(a-b).max():.1e}" for a,b in zip(r[2],o[2])))
rep("current (exact K1)", run(lambda l: ident))
rep("all layers fp16 x", run(lambda l: f16))
rep("layer0 exact, l>=1 fp16 x", run(lambda l: ident if l == 0 else f16))
print("max |h| per layer:", [float(np.abs(v).max()) for v in o[1]], "max |c|:", [float(np.abs(v).max()) for v in o[2]])
