#!/usr/bin/env python3
"""Small FAST/EXACT calls for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
  compute-sanitizer --tool racecheck python tools/sanitize.py
Exercises the list path (n<=16), the batched path (n>16), the verify path, the EXACT path and
the fallback (a flat row), at shapes small enough for the sanitizers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402


def main():
    ctx = api.Context(0)
    rng = np.random.default_rng(0)
    V, d, v_sub = 3000, 256, 2048
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16).float().cuda()
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    head = api.restrict_lm_head(ctx, W, api.RankedSubset(V, ids), dtype="bf16")
    for n in (4, 20):
        h = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
        h[1] = 0.0  # flat row -> fallback
        for mode in ("fast", "exact"):
            api.draft_head_topk(ctx, h, head, 8, mode=mode)
    hv = torch.from_numpy(rng.standard_normal((5, d)).astype(np.float32)).cuda()
    api.verify_head_argmax(ctx, hv, W.to(torch.bfloat16), mode="fast")
    api.verify_head_argmax(ctx, hv, W, mode="exact")
    # the draft layer (staged exact GEMV with a K tail chunk, tree attention, norms, RoPE, SiLU)
    dm, heads, Vm = 264, 4, 500
    wt = lambda r, c: (rng.standard_normal((r, c)) * 0.05).astype(np.float32)  # noqa: E731
    model = api.DraftModel(ctx, {"embedding": wt(Vm, dm), "wq": wt(dm, dm), "wk": wt(dm, dm), "wv": wt(dm, dm),
                                 "wo": wt(dm, dm), "w_up": wt(4 * dm, dm), "w_down": wt(dm, 4 * dm)}, heads, 256)
    model.forward(rng.integers(0, Vm, 70), np.arange(70), np.tril(np.ones((70, 70), np.uint8)))
    allow = np.zeros((3, 73), np.uint8)
    allow[:, :70] = 1
    allow[np.arange(3), 70 + np.arange(3)] = 1
    model.forward(rng.integers(0, Vm, 3), np.full(3, 70), allow)
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
