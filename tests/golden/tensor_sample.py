"""Which entries of a full-size forward the tensor goldens store.

The BASELINE configs c2-c5 produce y tensors of 32 MiB to 2 GiB, too large to
commit.  Each golden keeps the final states of every layer-direction and y at
three timesteps, for a fixed subset of batch rows (all rows up to 64; above
that the first 32 rows — one rank of c5's 8-way request shard — plus four rows
spread over the rest).  Shared by make_tensor_golden.py (writer) and the GPU
parity tests (reader), so both index the same entries.
"""
from __future__ import annotations


def sample_index(T: int, B: int) -> tuple[list[int], list[int]]:
    ts = sorted({0, T // 2, T - 1})
    if B <= 64:
        bs = list(range(B))
    else:
        bs = list(range(32)) + [B // 4 - 1, B // 2 - 1, 3 * B // 4 - 1, B - 1]
    return ts, bs


def take(y, hn, cn, T: int, B: int):
    """(y[ts][:, bs], hn[:, bs], cn[:, bs]) for numpy arrays or torch tensors."""
    ts, bs = sample_index(T, B)
    ys = y[ts][:, bs]
    hs = hn[:, bs]
    cs = None if cn is None else cn[:, bs]
    return ys, hs, cs
