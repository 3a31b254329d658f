#!/usr/bin/env python3
"""One draft-layer forward at the Llama-3-8B shape (10 rows, 512-row cache): for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402

d, heads, V, n, ctx_len = 4096, 32, 32000, 10, 512
ctx = api.Context(0)
rs = np.random.default_rng(0)
w = lambda r, c: (rs.standard_normal((r, c)) * 0.02).astype(np.float32)  # noqa: E731
model = api.DraftModel(ctx, {"embedding": w(V, d), "wq": w(d, d), "wk": w(d, d), "wv": w(d, d), "wo": w(d, d),
                             "w_up": w(4 * d, d), "w_down": w(d, 4 * d)}, heads, 1024)
model.forward(rs.integers(0, V, ctx_len), np.arange(ctx_len), np.tril(np.ones((ctx_len, ctx_len), np.uint8)))
allow = np.zeros((n, ctx_len + n), np.uint8)
allow[:, :ctx_len] = 1
allow[np.arange(n), ctx_len + np.arange(n)] = 1
for _ in range(2):
    model.truncate(ctx_len)
    model.forward(rs.integers(0, V, n), np.full(n, ctx_len), allow)
torch.cuda.synchronize()
print("ok")
import time  # noqa: E402
toks = rs.integers(0, V, n)
for trial in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        model.truncate(ctx_len)
        model.forward(toks, np.full(n, ctx_len), allow)
    torch.cuda.synchronize()
    print("forward ms", round((time.perf_counter() - t0) * 1000 / 5, 3), flush=True)
