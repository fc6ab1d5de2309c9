"""ctypes declarations mirroring include/sidp.h (argument marshalling only).

Loading fails loudly if libsidp.so is missing: there is no CPU fallback anywhere in the
product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SIDP_LIB: another build of the same library (A/B experiments between builds on one box)
LIB_PATH = os.environ.get("SIDP_LIB") or os.path.join(HERE, "libsidp.so")

SIDP_OK, SIDP_EINVAL, SIDP_ECUDA, SIDP_ENOMEM, SIDP_ESTATE, SIDP_EPEER, SIDP_ETIMEOUT = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "SIDP_OK", -1: "SIDP_EINVAL", -2: "SIDP_ECUDA", -3: "SIDP_ENOMEM",
                -4: "SIDP_ESTATE", -5: "SIDP_EPEER", -6: "SIDP_ETIMEOUT"}
WAS, CAS, REPLICATED = 0, 1, 2
ORDER_EXEC, ORDER_PAPER = 0, 1
POOL_LAYER, POOL_FFN = 0, 1
FETCH_SM, FETCH_CE = 0, 1


class ModelDesc(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("hidden", C.c_int32), ("n_q_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("intermediate", C.c_int32),
                ("vocab", C.c_int32), ("qkv_bias", C.c_int32), ("qk_norm", C.c_int32),
                ("rms_eps", C.c_float), ("rope_theta", C.c_float)]


class Config(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("layer_owner", C.POINTER(C.c_int32)),
                ("was_slots", C.c_int32), ("cas_slots", C.c_int32), ("order", C.c_int32),
                ("pool_scope", C.c_int32), ("max_batch", C.c_int32), ("max_ctx", C.c_int32),
                ("fetch_sms", C.c_int32), ("fetch_engine", C.c_int32), ("stagger", C.c_int32),
                ("device", C.c_int32), ("seed", C.c_uint64), ("fetch_pace_gbps", C.c_float),
                ("compute_sms", C.c_int32), ("slot_parts", C.c_int32),
                ("fetch_ce_share", C.c_float)]


class KV(C.Structure):
    _fields_ = [("k_cache", C.c_void_p), ("v_cache", C.c_void_p), ("pos", C.c_void_p),
                ("max_pos", C.c_int32), ("block_table", C.c_void_p), ("block_tokens", C.c_int32),
                ("max_blocks", C.c_int32), ("num_blocks", C.c_int32)]


class Batch(C.Structure):
    _fields_ = [("tokens", C.c_void_p), ("next", C.c_void_p), ("batch", C.c_int32), ("kv", KV),
                ("logits", C.c_void_p), ("layer_inputs", C.c_void_p), ("pos_out", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("fetches", C.c_uint64), ("bytes_fetched", C.c_uint64),
                ("launches", C.c_uint64), ("cas_round_trips", C.c_uint64), ("mode", C.c_int32),
                ("timeouts", C.c_int32), ("layer_bytes", C.c_uint64),
                ("local_layer_bytes", C.c_uint64), ("owned_bytes", C.c_uint64),
                ("slot_bytes", C.c_uint64), ("replicated_bytes", C.c_uint64),
                ("workspace_bytes", C.c_uint64), ("timed_ms", C.c_double * 8),
                ("timed_launches", C.c_uint64 * 8), ("fetch_sms_held", C.c_int32),
                ("compute_sms", C.c_int32), ("stagger_tick_ns", C.c_double),
                ("graph_replays", C.c_uint64), ("slot_checks", C.c_uint64),
                ("slot_mismatches", C.c_uint64)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_PI32 = C.POINTER(C.c_int32)

SIGNATURES = {
    "sidp_init": [C.POINTER(ModelDesc), C.POINTER(Config), C.POINTER(_P)],
    "sidp_alloc": [_P],
    "sidp_owned_bytes": [_P, C.POINTER(C.c_uint64)],
    "sidp_alloc_owned": [_P, _P, C.c_uint64],
    "sidp_alloc_serve_only": [_P],
    "sidp_alloc_serve_only_alias": [_P, _P],
    "sidp_init_weights_synthetic": [_P, _P],
    "sidp_export_handles": [_P, _P, C.POINTER(C.c_size_t)],
    "sidp_import_handles": [_P, C.POINTER(_P), C.POINTER(C.c_size_t)],
    "sidp_destroy": [_P],
    "sidp_decode_layer": [_P, _P, _I32, _I32, _I32, C.POINTER(KV), _P],
    "sidp_step": [_P, C.POINTER(Batch), _P],
    "sidp_set_mode": [_P, _I32, _I64],
    "sidp_set_batches": [_P, _PI32],
    "sidp_owner_of": [_P, _I32, _PI32],
    "sidp_get_plan": [_P, _PI32, _I32, _PI32],
    "sidp_get_schedule": [_P, _I32, _PI32, _PI32, _PI32, _I32, _PI32],
    "sidp_stagger_ticks": [_P, _PI32],
    "sidp_get_fetch_log": [_P, _PI32, _PI32, _PI32, _I32, _PI32],
    "sidp_get_fetch_trace": [_P, C.POINTER(_I64), _I32, _PI32],
    "sidp_get_consume_log": [_P, C.POINTER(_I64), _I32, _PI32],
    "sidp_stats": [_P, C.POINTER(Stats)],
    "sidp_set_timing": [_P, _I32],
    "sidp_last_error": [],
    "sidp_test_gemm": [_P, _I32, _P, _I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _I32, _P, _I32, _P],
    "sidp_test_gemm_qkv": [_P, _I32, _P, _I32, _I32, _P, _I32, _I32, _I32, _P, _P, C.c_float, _P,
                           _P, _P, _P, _P, _I32, _I32, _P],
    "sidp_test_gemm_resid_norm": [_P, _I32, _P, _I32, _I32, _I32, _P, _I32, _P, C.c_float, _P,
                                  _P, _P],
    "sidp_test_mlp_fused": [_P, _P, _P, _P, _I32, _I32, _I32, _P, C.c_float, _P, _P, _P, _P],
    "sidp_test_mlp_schedule": [_I32, _I32, _I32, _I32, _I32, _I32, _I32, _PI32, _I32, _PI32, _PI32,
                               _PI32],
    "sidp_test_gen": [_P, _I64, _I64, _I64, C.c_uint64, _I32, _I32, _I32, _I32, _I64, _I64, _I32, _P],
    "sidp_test_gen_kv": [_P, _I32, _I32, _I32, _I32, _I32, _I64, C.c_uint64, _I32, _I32, _P],
    "sidp_layer_ptr": [_P, _I32, C.POINTER(_P), C.POINTER(_P)],
    "sidp_debug_flags": [_P, C.POINTER(C.c_uint64), _I32],
    "sidp_test_fetch": [_P, _P, C.c_size_t, _I32, _I32, _P],
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libsidp.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            if name == "sidp_last_error":
                f.restype = C.c_char_p
            elif name == "sidp_destroy":
                f.restype = None
            else:
                f.restype = C.c_int
        _lib = L
    return _lib


class SidpError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().sidp_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(status: int, where: str):
    if status != SIDP_OK:
        raise SidpError(status, where)
