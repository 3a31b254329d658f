#!/usr/bin/env python3
"""FAST draft-head diagnostics on one GPU: per-call device time (CUDA events on the launch
stream), certification outcome and fallback reasons over many random C2 inputs.

  python tools/fast_diag.py [--calls 400] [--v-sub 32768] [--rows 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402
from paper_2502_14856_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=400)
    ap.add_argument("--v-sub", type=int, default=32768)
    ap.add_argument("--rows", type=int, default=10)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=128256)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(a.vocab, a.d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(a.vocab).astype(np.int32)
    subset = api.subset_from_ranking(ranked, a.v_sub, a.vocab, forced=[0, 1])
    head = api.restrict_lm_head(ctx, W, subset, dtype="bf16")
    del W
    gh = torch.Generator(device=dev).manual_seed(7)
    hs = [torch.randn(a.rows, a.d, generator=gh, device=dev) for _ in range(a.calls)]
    hs = [(x * torch.rsqrt(x.double().pow(2).mean(1, keepdim=True) + 1e-5).float()).contiguous() for x in hs]
    out = api.draft_head_topk(ctx, hs[0], head, 10, mode="fast")
    for i in range(10):
        api.draft_head_topk(ctx, hs[i], head, 10, mode="fast", out=out)
    torch.cuda.synchronize()
    times, rec_times, flags_all = [], [], []
    s = torch.cuda.current_stream()
    for x in hs:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        api.draft_head_topk(ctx, x, head, 10, mode="fast", out=out)
        e1.record(s)
        e1.synchronize()
        f = out.flags.cpu().numpy()
        flags_all.append(f)
        (rec_times if (f & _lib.FLAG_RECOMPUTED).any() else times).append(e0.elapsed_time(e1) * 1000)
    F = np.concatenate(flags_all)
    ns = (F >> 8) & 0xff
    cert = (F & _lib.FLAG_RECOMPUTED) == 0
    res = {
        "v_sub": a.v_sub, "rows": a.rows, "calls": a.calls,
        "us_certified_calls": {"median": float(np.median(times)) if times else None,
                               "p10": float(np.percentile(times, 10)) if times else None,
                               "p90": float(np.percentile(times, 90)) if times else None, "n": len(times)},
        "us_fallback_calls": {"median": float(np.median(rec_times)) if rec_times else None, "n": len(rec_times)},
        "rows_total": int(F.size), "rows_recomputed": int(((F & _lib.FLAG_RECOMPUTED) != 0).sum()),
        "reason_tie": int(((F & 0x10) != 0).sum()), "reason_bound": int(((F & 0x20) != 0).sum()),
        "reason_overflow": int(((F & 0x40) != 0).sum()),
        "slab_bytes": a.v_sub * a.d * 2,
        "cand_set_size": {"mean": float(ns[cert].mean()), "p50": float(np.median(ns[cert])),
                          "p99": float(np.percentile(ns[cert], 99)), "max": int(ns[cert].max())},
    }
    med = res["us_certified_calls"]["median"]
    if med:
        res["GBps_certified_median"] = a.v_sub * a.d * 2 / (med * 1e-6) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
