"""ctypes binding of libhobbit.so (include/hobbit.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels / C++ host code.

There is no fallback: if the shared library is missing or a symbol is absent
this module raises at import time, and every call that returns an HB_E* code
raises HobbitError with the library's message.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# HOBBIT_LIB: an alternative in-tree build (kernel-variant experiments only)
LIB_PATH = os.environ.get("HOBBIT_LIB") or os.path.join(PKG, "libhobbit.so")
HEADER = os.path.join(ROOT, "include", "hobbit.h")

HB_OK, HB_EINVAL, HB_ECAPACITY, HB_ESTATE, HB_ECUDA, HB_ENOMEM, HB_EUNSUPPORTED, HB_ENCCL = \
    0, -1, -2, -3, -4, -5, -6, -7
ERR_NAMES = {-1: "HB_EINVAL", -2: "HB_ECAPACITY", -3: "HB_ESTATE", -4: "HB_ECUDA",
             -5: "HB_ENOMEM", -6: "HB_EUNSUPPORTED", -7: "HB_ENCCL"}
HB_F16, HB_Q8, HB_Q4, HB_Q2 = 0, 1, 2, 3
HB_HIGH, HB_LOW, HB_SKIP = 0, 1, 2
HB_ENC_NONE = 255
HB_REG_DEVICE_BORROW, HB_REG_HOST_PINNED, HB_REG_HOST_COPY, HB_REG_DEVICE_COPY = 1, 2, 3, 4
HB_REG_CANONICAL = 0x100


class HobbitError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class hb_config(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("n_experts", C.c_int), ("top_k", C.c_int),
                ("hidden", C.c_int), ("ffn", C.c_int), ("hi_enc", C.c_int), ("lo_enc", C.c_int),
                ("t1", C.c_double), ("t2", C.c_double), ("lookahead_p", C.c_int),
                ("w_lru", C.c_int), ("w_lfu", C.c_int), ("w_lhu", C.c_int), ("w_fld", C.c_int),
                ("cap_high", C.c_int), ("cap_low", C.c_int), ("allow_upgrade", C.c_int),
                ("rank", C.c_int), ("world", C.c_int), ("max_batch", C.c_int),
                ("strict", C.c_int), ("device_cache", C.c_int), ("token_sharded", C.c_int),
                ("prefetch_both", C.c_int), ("deterministic", C.c_int)]


class hb_decision(C.Structure):
    _fields_ = [("token", C.c_int32), ("expert", C.c_int32), ("sel_rank", C.c_uint8),
                ("prec", C.c_uint8), ("served_enc", C.c_uint8), ("hit", C.c_uint8),
                ("gate", C.c_float)]


class hb_event(C.Structure):
    _fields_ = [("type", C.c_int32), ("kind", C.c_int32), ("layer", C.c_int32),
                ("expert", C.c_int32), ("enc", C.c_int32), ("slot", C.c_int32),
                ("victim", C.c_int32)]

    def as_tuple(self):
        return (self.type, self.kind, self.layer, self.expert, self.enc, self.slot, self.victim)


_P = C.c_void_p
_SIGS = {
    "hb_config_default": (None, [C.POINTER(hb_config)]),
    "hb_blob_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "hb_blob_section": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "hb_canonical_section": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "hb_repack_canonical": (C.c_int, [C.c_int, C.c_int, C.c_int, _P, _P, _P]),
    "hb_theta": (C.c_int64, [C.c_double, C.POINTER(C.c_int)]),
    "hb_last_error": (C.c_char_p, [_P]),
    "hb_version": (C.c_char_p, []),
    "hb_create": (C.c_int, [C.POINTER(hb_config), C.c_int, C.POINTER(_P)]),
    "hb_destroy": (C.c_int, [_P]),
    "hb_set_router": (C.c_int, [_P, C.c_int, _P, C.c_int]),
    "hb_register_expert": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, C.c_size_t, C.c_int]),
    "hb_token_begin": (C.c_int, [_P]),
    "hb_reset_sequence": (C.c_int, [_P]),
    "expert_cache_load": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P]),
    "prefetch_next_layer": (C.c_int, [_P, C.c_int, _P, C.c_int, _P]),
    "moe_layer_forward": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P]),
    "hb_get_decisions": (C.c_int, [_P, C.POINTER(hb_decision), C.c_int]),
    "hb_get_logits": (C.c_int, [_P, C.POINTER(C.c_int64), C.c_int]),
    "hb_get_events": (C.c_int, [_P, C.POINTER(hb_event), C.c_int]),
    "hb_last_expert_bytes": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "hb_copy_stats": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "hb_ts_buffer_bytes": (C.c_int, [_P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                     C.POINTER(C.c_size_t)]),
    "hb_ts_dispatch": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P, _P]),
    "hb_ts_compute": (C.c_int, [_P, C.c_int, _P, _P, _P, _P]),
    "hb_ts_combine": (C.c_int, [_P, _P, C.c_int, _P, _P]),
    "hb_launch_count": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "hb_set_batched_min": (C.c_int, [_P, C.c_int]),
    "hb_nccl_unique_id": (C.c_int, [_P]),
    "hb_nccl_init": (C.c_int, [_P, _P]),
    "hb_ep_broadcast_x": (C.c_int, [_P, _P, C.c_int, C.c_int, _P]),
    "hb_nccl_init_ranks": (C.c_int, [_P, _P, C.c_int, C.c_int]),
    "hb_profile": (C.c_int, [_P, C.c_int]),
    "hb_profile_read": (C.c_int, [_P, C.POINTER(C.c_float), C.c_int]),
    "hb_stamps": (C.c_int, [_P, C.c_int]),
    "hb_stamps_read": (C.c_int, [_P, C.POINTER(C.c_uint64), C.c_int]),
    "hb_quantize_expert": (C.c_int, [C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, _P]),
    "hb_synth_fill_f16": (C.c_int, [_P, C.c_size_t, C.c_uint64, C.c_float, C.c_uint64, _P]),
    "hbc_create": (C.c_int, [C.POINTER(hb_config), C.POINTER(_P)]),
    "hbc_destroy": (C.c_int, [_P]),
    "hbc_token_begin": (C.c_int, [_P]),
    "hbc_reset_sequence": (C.c_int, [_P]),
    "hbc_forward": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_uint8),
                              C.POINTER(C.c_uint8)]),
    "hbc_prefetch": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_uint8),
                               C.POINTER(C.c_int)]),
    "hbc_load": (C.c_int, [_P, C.c_int, C.c_int, C.c_int]),
    "hbc_get_events": (C.c_int, [_P, C.POINTER(hb_event), C.c_int]),
    "hbc_last_error": (C.c_char_p, [_P]),
}


def header_symbols():
    """Every function name declared in include/hobbit.h."""
    with open(HEADER) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(\w+)\s*\(", text, flags=re.M)))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run python -m paper_2411_01433_b200.build "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)          # AttributeError if not exported
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(code, ctx=None):
    if code is not None and code < 0:
        raise HobbitError(code, lib.hb_last_error(ctx).decode())
    return code


def default_config(**kw) -> hb_config:
    cfg = hb_config()
    lib.hb_config_default(C.byref(cfg))
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise KeyError(k)
        setattr(cfg, k, v)
    return cfg


def blob_bytes(enc, hidden, ffn) -> int:
    return int(lib.hb_blob_bytes(enc, hidden, ffn))


def blob_section(enc, hidden, ffn, mat, sec):
    off, nb = C.c_size_t(), C.c_size_t()
    check(lib.hb_blob_section(enc, hidden, ffn, mat, sec, C.byref(off), C.byref(nb)))
    return off.value, nb.value


def canonical_section(enc, hidden, ffn, mat, sec):
    off, nb = C.c_size_t(), C.c_size_t()
    check(lib.hb_canonical_section(enc, hidden, ffn, mat, sec, C.byref(off), C.byref(nb)))
    return off.value, nb.value


def theta(t: float):
    kind = C.c_int()
    v = lib.hb_theta(t, C.byref(kind))
    return None if kind.value > 0 else (-(1 << 200) if kind.value < 0 else int(v))
