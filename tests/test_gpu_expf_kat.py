"""Exhaustive known-answer test of the device glibc expf ports:
every float in [-104, 0] (1,120,927,745 bit patterns from -0.0 to -104.0, the whole softmax
input domain x = l - max <= 0), plus +0.0, through both device ports — the branchy
dev::expf_glibc and the branch-free dev::expf_glibc_nb — against the host libm's expf on the
same machine. Zero mismatches required."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import _lib

pytestmark = pytest.mark.gpu

FIRST, LAST = 0x80000000, 0xC2D00000  # -0.0 .. -104.0


def run_range(ctx, restatement, first, count, corrupt=None):
    host = restatement.libm_expf_range(first, count)
    if corrupt is not None:
        host[corrupt] = np.nextafter(host[corrupt], np.float32(2.0))
    exp_dev = torch.from_numpy(host).cuda()
    out = torch.tensor([0, 0, -1, -1], dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().frs_debug_expf_check(ctx.handle, first, count, C.c_void_p(exp_dev.data_ptr()),
                                               C.c_void_p(out.data_ptr()), None), "expf check")
    torch.cuda.synchronize()
    o = out.cpu().numpy().view(np.uint64)
    return int(o[0]), int(o[1]), int(o[2]), int(o[3])


def test_expf_ports_exhaustive(cuda_ctx, restatement):
    # the check is live: one corrupted expected value is reported by both ports, at its index
    assert run_range(cuda_ctx, restatement, FIRST + 12345, 1 << 20, corrupt=777) == (1, 1, 777, 777)
    total = LAST - FIRST + 1
    assert total == 1120927745
    chunk = 1 << 27
    for start in range(0, total, chunk):
        n = min(chunk, total - start)
        b0, b1, f0, f1 = run_range(cuda_ctx, restatement, FIRST + start, n)
        assert b0 == 0, f"expf_glibc: {b0} mismatches, first at bits {FIRST + start + f0:#x}"
        assert b1 == 0, f"expf_glibc_nb: {b1} mismatches, first at bits {FIRST + start + f1:#x}"
    assert run_range(cuda_ctx, restatement, 0, 1)[:2] == (0, 0)  # +0.0


def test_expf_ports_specials(cuda_ctx, restatement):
    """Outside the softmax domain: positive arguments up to overflow, -inf / +inf / NaN."""
    for first, count in ((0x3F800000, 1 << 20), (0x42B00000, 1 << 16), (0xFF800000, 1), (0x7F800000, 1),
                         (0xC2D00000, 1 << 16)):
        b0, b1, _, _ = run_range(cuda_ctx, restatement, first, count)
        assert (b0, b1) == (0, 0), hex(first)
