#!/usr/bin/env python3
"""C5 (256 independent decode streams) cost split at C2: one decode_step_table_multi iteration
against its two device-heavy parts timed alone — the EXACT draft level over S x width rows and
the FAST verify head over S x 61 rows (CUDA events). Diagnostic.

  python tools/streams_probe.py [S]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    d, V, v_sub = 4096, 128256, 32768
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    sub = api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1])
    dh = api.DeviceHead(ctx, W, sub, dtype="bf16")
    head = api.restrict_lm_head(ctx, W, sub, dtype="bf16")
    E = torch.randn(V, d, generator=g, device=dev)
    E = E * torch.rsqrt((E.double() ** 2).mean(1, keepdim=True) + 1e-5).float()
    Wb = W.to(torch.bfloat16)
    del W
    params = api.DraftParams(10, 6, 60)
    roots = [int(x) for x in np.random.default_rng(7).integers(0, V, S)]
    res = api.decode_step_table_multi(dh, E, roots, Wb, params, mode="fast")
    roots = [int(o.emitted[-1]) for _, o in res]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = api.decode_step_table_multi(dh, E, roots, Wb, params, mode="fast")
    it_ms = 1000 * (time.perf_counter() - t0)
    rows = E[torch.randint(0, V, (S * 10,), device=dev, generator=g)]
    lvl_ms = timed(lambda: api.draft_head_topk(ctx, rows, head, 10, mode="exact", want_total=False))
    lvl0_ms = timed(lambda: api.draft_head_topk(ctx, rows[:S], head, 10, mode="exact", want_total=False))
    vrows = E[torch.randint(0, V, (S * 61,), device=dev, generator=g)]
    ver_ms = timed(lambda: api.verify_head_argmax(ctx, vrows, Wb, mode="fast"))
    print({"streams": S, "iteration_ms": round(it_ms, 2), "exact_level_ms_S_x_10_rows": round(lvl_ms, 2),
           "exact_level_ms_S_rows": round(lvl0_ms, 2), "fast_verify_ms_S_x_61_rows": round(ver_ms, 2),
           "device_estimate_ms": round(lvl0_ms + 5 * lvl_ms + ver_ms, 2),
           "tokens": sum(o.accepted_length() for _, o in res)})


if __name__ == "__main__":
    main()
