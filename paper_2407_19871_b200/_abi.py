"""ctypes binding of the C ABI in include/locpir_b200.h.

This is the binding a maintainer of the reference would add to reach the B200
engine from Python.  There is no fallback: if the in-tree
library paper_2407_19871_b200/liblocpir_b200.so is missing, importing the
package raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# LOCPIR_B200_LIB selects an alternative in-tree build (A/B experiments)
LIB_PATH = os.environ.get("LOCPIR_B200_LIB") or os.path.join(HERE, "liblocpir_b200.so")

OK, EINVAL, ELOGIC, ECUDA, ENOMEM = 0, -1, -2, -3, -4
AND, OR, XOR, XNOR, NAND, MUX, NOT, NOR, COPY, CONST, ANDNY, ORNY, MAJ, XOR3 = range(14)
SLOT_NONE = 0xFFFFFFFF


class Params(C.Structure):
    _fields_ = [("n", C.c_uint32), ("N", C.c_uint32), ("k", C.c_uint32),
                ("bk_l", C.c_uint32), ("bk_bgbit", C.c_uint32), ("ks_t", C.c_uint32),
                ("ks_basebit", C.c_uint32), ("alpha_in", C.c_double), ("alpha_bk", C.c_double)]


class GateOp(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("in0", C.c_uint32), ("in1", C.c_uint32),
                ("in2", C.c_uint32), ("out", C.c_uint32)]


# (name, restype, argtypes) -- every symbol declared in include/locpir_b200.h
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_P = C.POINTER(Params)
_ops = C.POINTER(GateOp)
_ctx = C.c_void_p
SIGNATURES = [
    ("locpir_b200_params_default", C.c_int, [C.c_int, _P]),
    ("locpir_b200_bk_words", C.c_size_t, [_P]),
    ("locpir_b200_ksk_words", C.c_size_t, [_P]),
    ("locpir_b200_keygen", C.c_int, [_P, C.c_uint64, _u8p, _u8p, _u32p, _u32p]),
    ("locpir_b200_keygen_with_lwe_key", C.c_int, [_P, C.c_uint64, _u8p, _u8p, _u32p, _u32p]),
    ("locpir_b200_encrypt_bits", C.c_int, [_P, _u8p, C.c_uint64, _u8p, C.c_uint64, _u32p]),
    ("locpir_b200_decrypt_bits", C.c_int, [_P, _u8p, _u32p, C.c_uint64, _u8p]),
    ("locpir_b200_ctx_create", C.c_int, [_P, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("locpir_b200_ctx_destroy", None, [_ctx]),
    ("locpir_b200_last_error", C.c_char_p, [_ctx]),
    ("locpir_b200_stream", C.c_void_p, [_ctx]),
    ("locpir_b200_upload_keys", C.c_int, [_ctx, C.c_void_p, C.c_void_p, C.c_int]),
    ("locpir_b200_pool_reserve", C.c_int, [_ctx, C.c_uint64]),
    ("locpir_b200_pool_capacity", C.c_uint64, [_ctx]),
    ("locpir_b200_pool_h2d", C.c_int, [_ctx, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("locpir_b200_pool_d2h", C.c_int, [_ctx, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("locpir_b200_pool_load_device", C.c_int, [_ctx, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("locpir_b200_pool_store_device", C.c_int, [_ctx, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("locpir_b200_run", C.c_int, [_ctx, _ops, C.c_uint64]),
    ("locpir_b200_eval_level", C.c_int, [_ctx, _ops, C.c_uint64]),
    ("locpir_b200_sync", C.c_int, [_ctx]),
    ("locpir_b200_program_create", C.c_int, [_ctx, _ops, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("locpir_b200_program_launch", C.c_int, [_ctx, C.c_void_p]),
    ("locpir_b200_program_prepare", C.c_int, [_ctx, C.c_void_p]),
    ("locpir_b200_program_kernels", C.c_uint64, [C.c_void_p]),
    ("locpir_b200_program_destroy", None, [C.c_void_p]),
    ("locpir_b200_plan", C.c_int, [_ops, C.c_uint64, _u32p, _u64p, _u64p]),
    ("locpir_b200_counters", C.c_int, [_ctx, _u64p]),
    ("locpir_b200_counters_reset", C.c_int, [_ctx]),
    ("locpir_b200_gate_batch_host", C.c_int,
     [_ctx, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
    ("locpir_b200_loc_pir_scratch", C.c_uint64, [C.c_uint32] * 4),
    ("locpir_b200_loc_pir", C.c_int,
     [_ctx, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p, _u32p, _u32p, _u32p,
      C.c_uint64, C.c_int]),
    ("locpir_b200_loc_pir_program", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p, _u32p, _u32p, _u32p,
      C.c_uint64, C.c_int, _ops, _u64p]),
    ("locpir_b200_loc_pir_maj_program", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p, _u32p, _u32p, _u32p,
      C.c_uint64, C.c_int, _ops, _u64p]),
    ("locpir_b200_loc_pir_program_ex", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p, _u32p, C.POINTER(C.c_int64),
      _u32p, _u32p, C.c_uint64, C.c_int, C.c_int, _ops, _u64p]),
    ("locpir_b200_loc_pir_folded_scratch", C.c_uint64, [C.c_uint32] * 4),
    ("locpir_b200_loc_pir_folded_program", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p, C.POINTER(C.c_int64), _u32p,
      _u32p, C.c_uint64, C.c_int, _ops, _u64p]),
    ("locpir_b200_check_query_payload", C.c_int,
     [_P, C.c_void_p, C.c_uint64, C.c_uint32, C.c_char_p, C.c_uint64]),
    ("locpir_b200_pool_load_queries", C.c_int,
     [_ctx, C.c_void_p, _u64p, C.c_uint64, C.c_uint32, _u32p, _u32p]),
    ("locpir_b200_pool_load_zero_sheet", C.c_int,
     [_ctx, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p, C.c_uint32]),
    ("locpir_b200_pool_store_responses", C.c_int,
     [_ctx, _u32p, C.c_uint64, C.c_uint32, C.c_void_p]),
    ("locpir_b200_server_create", C.c_int,
     [_ctx, C.POINTER(C.c_int64), _u64p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
      C.POINTER(C.c_void_p)]),
    ("locpir_b200_server_create_at", C.c_int,
     [_ctx, C.c_uint64, C.POINTER(C.c_int64), _u64p, C.c_uint32, C.c_uint32, C.c_uint32,
      C.c_uint32, C.c_int, C.POINTER(C.c_void_p)]),
    ("locpir_b200_server_destroy", None, [C.c_void_p]),
    ("locpir_b200_server_last_error", C.c_char_p, [C.c_void_p]),
    ("locpir_b200_server_open_session", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32)]),
    ("locpir_b200_server_close_session", C.c_int, [C.c_void_p, C.c_uint32]),
    ("locpir_b200_server_submit", C.c_int,
     [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    ("locpir_b200_server_pending", C.c_uint64, [C.c_void_p]),
    ("locpir_b200_server_flush", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    ("locpir_b200_server_take_response", C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    ("locpir_b200_client_encrypt", C.c_int,
     [_ctx, _u8p, C.c_uint64, C.c_uint32, _u32p, C.c_uint64, C.c_uint64]),
    ("locpir_b200_debug_blind_rotate", C.c_int, [_ctx, C.c_void_p, C.c_uint64, C.c_void_p]),
    ("locpir_b200_debug_fft_error", C.c_int,
     [_ctx, C.c_void_p, C.c_uint64, C.POINTER(C.c_double)]),
    ("locpir_b200_debug_keyswitch", C.c_int, [_ctx, C.c_void_p, C.c_uint64, C.c_void_p]),
    ("locpir_b200_timing_enable", C.c_int, [_ctx, C.c_int]),
    ("locpir_b200_kernel_stats", C.c_int, [_ctx, C.POINTER(C.c_double), _u64p]),
    ("locpir_b200_fp64_peak", C.c_int, [_ctx, C.POINTER(C.c_double)]),
]

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree CUDA library; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
