"""ctypes binding of libfrspec_cuda.so (include/frspec_cuda.h).

The product path has no CPU fallback: if the shared library is missing or cannot be
loaded, ``lib()`` raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FRS_LIB_PATH") or os.path.join(HERE, "libfrspec_cuda.so")  # override: A/B runs

FRS_OK, FRS_EINVAL, FRS_ECAPACITY, FRS_EDATA, FRS_ELOGIC, FRS_ECUDA, FRS_ENCCL, FRS_ENOTSUP = range(8)
DTYPE_F32, DTYPE_BF16 = 0, 1
MODE_EXACT, MODE_FAST = 0, 1
FLAG_NONFINITE, FLAG_SEQ_SUM, FLAG_UNCERTIFIED, FLAG_RECOMPUTED = 0x1, 0x2, 0x4, 0x8
FLAG_CERT_TIE, FLAG_CERT_BOUND, FLAG_CERT_OVERFLOW = 0x10, 0x20, 0x40
FLAG_SAMPLE_UNCERTIFIED = 0x80
FLAG_EMPTY_ROW = 0x100


class FrsError(RuntimeError):
    """Base of the C-ABI error mapping (frs_status)."""


class CapacityError(FrsError):
    """frspec::CapacityError (errors.h:10-12)."""


class DataError(FrsError):
    """frspec::DataError (errors.h:15-17)."""


class CudaError(FrsError):
    pass


class NotSupported(FrsError):
    pass


class InvalidArgument(FrsError, ValueError):
    """std::invalid_argument (errors.h:7)."""


class LogicError(FrsError):
    """std::logic_error / std::domain_error."""


_EXC = {FRS_EINVAL: InvalidArgument, FRS_ECAPACITY: CapacityError, FRS_EDATA: DataError,
        FRS_ELOGIC: LogicError, FRS_ECUDA: CudaError, FRS_ENCCL: FrsError, FRS_ENOTSUP: NotSupported}

# (name, restype, argtypes)
_P, _I, _I64, _F, _U64 = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_uint64
HIDDEN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                        C.c_void_p, C.c_void_p)
SIGNATURES = [
    ("frs_abi_version", _I, []),
    ("frs_last_error", C.c_char_p, []),
    ("frs_ctx_create", _I, [_I, C.POINTER(_P)]),
    ("frs_ctx_destroy", _I, [_P]),
    ("frs_ctx_sm_count", _I, [_P]),
    ("frs_ctx_reserve", _I, [_P, _I, _I64, _I]),
    ("frs_ctx_set_timing", _I, [_P, _I]),
    ("frs_ctx_timing_read", _I, [_P, C.POINTER(C.c_double), C.POINTER(_I)]),
    ("frs_ctx_launch_count", _I, [_P, C.POINTER(_U64)]),
    ("frs_debug_fast_partials", _I, [_P, _I, _I, _P, _P, _P, _P, _P]),
    ("frs_debug_expf_check", _I, [_P, C.c_uint32, _I64, _P, _P, _P]),
    ("frs_slab_build", _I, [_P, _P, _I64, _I, _P, _I, _I, _P, _P]),
    ("frs_slab_bytes", C.c_size_t, [_I, _I, _I]),
    ("frs_draft_head_topk", _I, [_P, _P, _I, _I, _P, _I, _I, _P, _I, _F, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("frs_slab_tile_bytes", C.c_size_t, [_I, _I]),
    ("frs_slab_tile", _I, [_P, _P, _I, _I, _P, _P]),
    ("frs_draft_head_topk_tiled", _I, [_P, _P, _I, _I, _P, _P, _I, _P, _I, _F, _P, _P, _P, _P, _P, _P, _P]),
    ("frs_verify_head_argmax_tiled", _I, [_P, _P, _I, _I, _P, _P, _I, _I, _P, _P, _P, _P]),
    ("frs_verify_head_argmax", _I, [_P, _P, _I, _I, _P, _I, _I, C.c_int32, _I, _P, _P, _P, _P]),
    ("frs_accept_greedy", _I, [_P, _P, _P, _P, _I, _P, _P, _P, _P]),
    ("frs_argmax_merge", _I, [_P, _P, _P, _I, _I, _P, _P, _P]),
    ("frs_gather_rows", _I, [_P, _P, _I64, _I, _P, _I, _P, _P]),
    ("frs_vocab_shard", _I, [_I64, _I, _I, C.POINTER(_I64), C.POINTER(_I64)]),
    ("frs_argmax_merge_host", _I, [_P, _P, _I, _I, _P, _P]),
    ("frs_count_frequencies", _I, [_P, _I64, _I, _P]),
    ("frs_build_subset", _I, [_P, _I, _I, _P, _I, _P]),
    ("frs_subset_from_ranking", _I, [_P, _I, _I, _I, _P, _I, _P]),
    ("frs_coverage", _I, [_P, _I, _P, _I, C.POINTER(C.c_double)]),
    ("frs_flops_ratio", _I, [_I, _I, C.POINTER(C.c_double)]),
    ("frs_tree_mask", _I, [_P, _I, _P]),
    ("frs_head_create", _I, [_P, _P, _I64, _I, _I, _P, _I, _I, C.POINTER(_P)]),
    ("frs_head_destroy", _I, [_P]),
    ("frs_head_info", _I, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    ("frs_head_draft_host", _I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    ("frs_draft_tree", _I, [_P, C.c_int32, HIDDEN_FN, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, C.POINTER(_I)]),
    ("frs_rng_create", _I, [C.c_uint64, C.POINTER(_P)]),
    ("frs_rng_destroy", _I, [_P]),
    ("frs_rng_uniforms", _I, [_P, _I, _P]),
    ("frs_draft_head_sample", _I, [_P, _P, _I, _I, _P, _I, _I, _P, _I, C.c_float, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("frs_count_frequencies_device", _I, [_P, _P, _I64, _I, _P, _P]),
    ("frs_draft_model_create", _I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.POINTER(_P)]),
    ("frs_draft_model_destroy", _I, [_P]),
    ("frs_draft_model_truncate", _I, [_P, _I]),
    ("frs_draft_model_length", _I, [_P, C.POINTER(_I)]),
    ("frs_draft_model_forward", _I, [_P, _P, _P, _I, _P, _P, _P]),
    ("frs_draft_model_position", _I, [_P, _I, C.POINTER(_I)]),
    ("frs_draft_model_compact", _I, [_P, _I, _P, _I, _P]),
    ("frs_draft_tree_model", _I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, C.POINTER(_I), _P, _P, _P]),
    ("frs_masked_attention", _I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P]),
    ("frs_write_token_stream", _I, [C.c_char_p, _I, _P, _I64]),
    ("frs_read_token_stream", _I, [C.c_char_p, _P, _I64, C.POINTER(_I), C.POINTER(_I64)]),
    ("frs_read_token_stream_text", _I, [C.c_char_p, _I, _P, _I64, C.POINTER(_I64)]),
    ("frs_write_ranked_file", _I, [C.c_char_p, _P, _I64]),
    ("frs_read_ranked_file", _I, [C.c_char_p, _P, _I64, C.POINTER(_I64)]),
    ("frs_verify_stochastic", _I, [_P, _P, _P, _I, _I, _I, _P, _P, _I, _P, _I, _P, _P, _P, C.c_float, _P, _P,
                                   C.POINTER(_I), _P, C.POINTER(_I)]),
    ("frs_draft_tree_sampled", _I, [_P, C.c_int32, HIDDEN_FN, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P,
                                    C.POINTER(_I), _P, _P, _P]),
    ("frs_verify_greedy", _I, [_P, _P, _P, _I, _I, _I, _I, _P, _P, _I, _P, C.POINTER(_I), _P, C.POINTER(_I)]),
    ("frs_verify_greedy_table", _I, [_P, _P, _I64, C.c_int32, _P, _I, _I, _I, _I, _P, _P, _I, _P, C.POINTER(_I), _P,
                                     C.POINTER(_I)]),
    ("frs_decode_step_table", _I, [_P, _P, C.c_int32, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, C.POINTER(_I),
                                   _P, C.POINTER(_I), _P, C.POINTER(_I)]),
    ("frs_decode_step_table_multi", _I, [_P, _P, _I, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P,
                                         _P, _P, _P]),
    ("frs_decode_step_table_tiled", _I, [_P, _P, C.c_int32, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P,
                                         C.POINTER(_I), _P, C.POINTER(_I), _P, C.POINTER(_I)]),
]



class AcceptanceStatsC(C.Structure):  # frs_acceptance_stats (include/frspec_cuda.h)
    HIST_MAX = 72
    _fields_ = [("iterations", C.c_int64), ("emitted", C.c_int64), ("mean_accepted_length", C.c_double),
                ("hist_len", C.c_int32), ("pad_", C.c_int32), ("histogram", C.c_int64 * 72)]


SIGNATURES += [
    ("frs_ctx_set_graphs", _I, [_P, _I]),
    ("frs_nccl_get_unique_id", _I, [_P]),
    ("frs_nccl_comm_init", _I, [_P, _I, _P, _I, C.POINTER(_P)]),
    ("frs_nccl_comm_destroy", _I, [_P]),
    ("frs_verify_head_argmax_vp", _I, [_P, _P, _P, _I, _I, _P, _I, _I, C.c_int32, _I, _P, _P, _P, _P]),
    ("frs_acceptance_add", _I, [C.POINTER(AcceptanceStatsC), _I]),
    ("frs_acceptance_merge", _I, [C.POINTER(AcceptanceStatsC), C.POINTER(AcceptanceStatsC)]),
    ("frs_accepted_length_stats", _I, [_P, _I, C.POINTER(AcceptanceStatsC)]),
]

_LIB = None


def lib() -> C.CDLL:
    """Load (once) and return the CUDA library. Raises if it is absent — no fallback."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2502_14856_b200.build` "
                              "(there is no CPU fallback for the FR-Spec hot path)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(status: int, what: str = "") -> None:
    if status != FRS_OK:
        msg = lib().frs_last_error().decode(errors="replace")
        raise _EXC.get(status, FrsError)(f"{what}: {msg}" if what else msg)
