#!/usr/bin/env python3
"""Exact GEMV (k_exact_gemv) timings at the shapes its consumers run: the C2 EXACT draft level
(V_sub 32768 x 4096 bf16 slab, n = 10), the draft layer's projections (4096 x 4096, 16384 x
4096, 4096 x 16384 fp32, n = 10), the verify head (128256 x 4096 bf16, n = 61). JSON lines:
device us per call (CUDA events over back-to-back calls; W > L2 or rotated copies)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402

PEAK = 6551.4


def timed(fn, iters=int(os.environ.get("ITERS", 50)), warm=3):
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / iters


def main():
    ctx = api.Context(0)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(7)
    for (rows, d, n, dt) in [(32768, 4096, 10, "bf16"), (4096, 4096, 10, "f32"), (16384, 4096, 10, "f32"),
                             (4096, 16384, 10, "f32"), (128256, 4096, 61, "bf16"), (32768, 4096, 1, "bf16"),
                             (32768, 4096, 32, "bf16")]:
        W = (torch.randn(rows, d, generator=g, device=dev) * 0.02)
        copies = max(1, (4 * 126 * 2 ** 20) // (rows * d * (2 if dt == "bf16" else 4)) + 1)
        heads = [api.restrict_lm_head(ctx, W, api.RankedSubset(rows, np.arange(rows, dtype=np.int32)), dtype=dt)
                 for _ in range(min(copies, 6))]
        h = torch.randn(n, d, generator=g, device=dev)
        out = api.draft_head_topk(ctx, h, heads[0], 1, mode="exact", want_logits=True)
        full = timed(lambda i: api.draft_head_topk(ctx, h, heads[i % len(heads)], 1, mode="exact", want_logits=True,
                                                   out=out))
        wbytes = rows * d * (2 if dt == "bf16" else 4)
        print(json.dumps(dict(rows=rows, d=d, n=n, dtype=dt, us_call=full, weight_gbs=wbytes / full / 1e3,
                              macs_per_s_T=rows * d * n / full / 1e6)), flush=True)
        del heads, W


if __name__ == "__main__":
    main()
