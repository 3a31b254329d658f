#!/usr/bin/env python3
"""Back-to-back FAST draft levels: device time per step (CUDA events around K steps) and host
enqueue time per step, with / without per-call timing events (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    d, V, v_sub, n = 4096, 128256, 32768, 10
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    head = api.restrict_lm_head(ctx, W, api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1]), dtype="bf16")
    del W
    pool = [torch.randn(n, d, generator=g, device=dev) for _ in range(16)]
    out = api.draft_head_topk(ctx, pool[0], head, 10, mode="fast")
    for i in range(40):
        api.draft_head_topk(ctx, pool[i % 16], head, 10, mode="fast", out=out)
    torch.cuda.synchronize()
    for timing in (False, True):
        ctx.set_timing(timing)
        K = 1000
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        t0 = time.perf_counter()
        for i in range(K):
            api.draft_head_topk(ctx, pool[i % 16], head, 10, mode="fast", out=out)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print(f"timing={timing}: device {e0.elapsed_time(e1) * 1000 / K:.1f} us/step, host enqueue "
              f"{(t1 - t0) * 1e6 / K:.1f} us/step", flush=True)
        if timing:
            ms, cnt = ctx.timing_read()
            print(f"   per-call events: {ms * 1000 / max(cnt, 1):.1f} us over {cnt} calls")
    # host cost of the python wrapper alone
    t0 = time.perf_counter()
    for i in range(1000):
        h = pool[i % 16].contiguous()
        _ = (h.data_ptr(), out.ridx.data_ptr(), out.full.data_ptr(), out.prob.data_ptr(), torch.cuda.current_stream().cuda_stream)
    print(f"python arg prep ~{(time.perf_counter() - t0) * 1e3:.1f} us/call")


if __name__ == "__main__":
    main()
