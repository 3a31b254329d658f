#!/usr/bin/env python3
"""Head-path decode loop at C2 (bench.py's decode measurement): wall time per decode_step_table
iteration; run under `ncu --metrics gpu__time_duration.sum` for the per-kernel split (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    d, V, v_sub = 4096, 128256, 32768
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    dh = api.DeviceHead(ctx, W, api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1]), dtype="bf16")
    E = torch.randn(V, d, generator=g, device=dev)
    E = E * torch.rsqrt((E.double() ** 2).mean(1, keepdim=True) + 1e-5).float()
    Wb = W.to(torch.bfloat16)
    del W
    params = api.DraftParams(10, 6, 60)
    token = 1
    for _ in range(3):
        token = int(api.decode_step_table(dh, E, token, Wb, params, mode=mode)[1].emitted[-1])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    acc = 0
    for _ in range(iters):
        _, out = api.decode_step_table(dh, E, token, Wb, params, mode=mode)
        acc += out.accepted_length()
        token = int(out.emitted[-1])
    dt = time.perf_counter() - t0
    print(f"decode_step_table: {dt * 1e3 / iters:.3f} ms/iter, {acc / dt:.1f} tokens/s, launches/iter "
          f"{ctx.launch_count / max(iters + 3, 1):.1f}")


if __name__ == "__main__":
    main()
