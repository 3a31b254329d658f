#!/usr/bin/env python3
"""C5 batched drafting: one call over `rows` hidden rows (256 streams x 10 beam rows = 2560 at
the Llama-3-8B shape), FAST head over the bf16 V_sub=32768 slab. Prints device us per call;
run under ncu for the per-kernel split."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2560
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    d, V, v_sub, k = 4096, 128256, 32768, 10
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    head = api.restrict_lm_head(ctx, W, api.RankedSubset(V, ranked[:v_sub]), dtype="bf16")
    del W
    h = torch.randn(rows, d, generator=g, device=dev)
    h = (h * torch.rsqrt(h.double().pow(2).mean(1, keepdim=True) + 1e-5).float()).contiguous()
    out = api.draft_head_topk(ctx, h, head, k, mode="fast")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        api.draft_head_topk(ctx, h, head, k, mode="fast", out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000.0 / iters
    print(json.dumps({"rows": rows, "us_per_call": us, "rows_per_s": rows / us * 1e6,
                      "recomputed": int(((out.flags & 0x8) != 0).sum().item())}))


if __name__ == "__main__":
    main()
