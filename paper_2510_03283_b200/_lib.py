"""ctypes binding of libmace_b200.so (the C-ABI declared in include/mace_b200.h).

There is deliberately no fallback: if the shared library is missing or no sm_100 device is present,
``Lib()`` / ``Ctx()`` raise. The product path never routes through torch math or the oracle.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
import os  # noqa: E402

# MACE_LIB selects an alternative in-tree build (e.g. the phase-traced GEMM of tools/gemm_trace.py)
LIB_PATH = _PKG / os.environ.get("MACE_LIB", "libmace_b200.so")


class MaceError(RuntimeError):
    pass


class MaceGemmArgs(C.Structure):
    _fields_ = [
        ("a", C.c_void_p), ("lda", C.c_int), ("a_mn_major", C.c_int),
        ("b", C.c_void_p), ("ldb", C.c_int), ("b_mn_major", C.c_int),
        ("M", C.c_int), ("N", C.c_int), ("K", C.c_int),
        ("out", C.c_void_p), ("ldo", C.c_int), ("mode", C.c_int),
        ("bias", C.c_void_p), ("alpha", C.c_float), ("split_k", C.c_int),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t), ("flags", C.c_int),
    ]


class MaceKvLayout(C.Structure):
    _fields_ = [
        ("ptab", C.c_void_p), ("max_prompt_pages", C.c_int),
        ("dtab", C.c_void_p), ("max_dec_pages", C.c_int),
        ("dec_base", C.c_void_p), ("dec_first", C.c_void_p), ("dec_end", C.c_void_p),
        ("free_stack", C.c_void_p), ("free_top", C.c_void_p), ("stack_cap", C.c_int),
        ("n_kv_heads", C.c_int), ("sink_page", C.c_int),
    ]


class MaceAttnArgs(C.Structure):
    _fields_ = [
        ("qkv", C.c_void_p), ("T", C.c_int), ("Hq", C.c_int), ("Hkv", C.c_int), ("hd", C.c_int),
        ("seqs", C.c_void_p),
        ("tc_items", C.c_void_p), ("n_tc", C.c_int),
        ("dec_items", C.c_void_p), ("n_dec", C.c_int),
        ("kv", MaceKvLayout),
        ("k_pool", C.c_void_p), ("v_pool", C.c_void_p), ("pool_pages", C.c_longlong),
        ("out", C.c_void_p), ("lse", C.c_void_p), ("head_norm", C.c_void_p),
        ("scale", C.c_float),
        ("dec_workspace", C.c_void_p), ("dec_workspace_bytes", C.c_size_t), ("dec_counters", C.c_void_p),
        ("dec_work", C.c_void_p), ("decode_impl", C.c_int), ("tc_pairs", C.c_int),
    ]


_LAYER_FIELDS = ("attn_norm_w", "attn_norm_b", "qkv_w", "qkv_b", "o_w", "o_b",
                 "mlp_norm_w", "mlp_norm_b", "up_w", "up_b", "down_w", "down_b")


class MaceLayerWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in _LAYER_FIELDS]


class MaceLayerGrads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in _LAYER_FIELDS]


class MaceLoraLayer(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("a_qkv", "a_o", "a_up", "a_down", "bt_o", "bt_down",
                                          "g_a_qkv", "g_a_o", "g_a_up", "g_a_down",
                                          "g_bt_qkv", "g_bt_o", "g_bt_up", "g_bt_down")]


class MaceModelDesc(C.Structure):
    _fields_ = [
        ("family", C.c_int), ("n_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int),
        ("n_kv_heads", C.c_int), ("head_dim", C.c_int), ("ffn", C.c_int), ("up_dim", C.c_int), ("vocab", C.c_int),
        ("norm_eps", C.c_float), ("dpo_beta", C.c_float),
        ("embed", C.c_void_p), ("pos_embed", C.c_void_p), ("final_norm_w", C.c_void_p), ("final_norm_b", C.c_void_p),
        ("layers", C.POINTER(MaceLayerWeights)),
        ("n_sel", C.c_int), ("sel_layers", C.POINTER(C.c_int)),
        ("ref_layers", C.POINTER(MaceLayerWeights)),
        ("ref_final_norm_w", C.c_void_p), ("ref_final_norm_b", C.c_void_p),
        ("grads", C.POINTER(MaceLayerGrads)),
        ("grad_final_norm_w", C.c_void_p), ("grad_final_norm_b", C.c_void_p),
        ("grad_flat", C.c_void_p), ("n_grad", C.c_longlong),
        ("cos_t", C.c_void_p), ("sin_t", C.c_void_p),
        ("kv", MaceKvLayout),
        ("k_pool", C.c_void_p), ("v_pool", C.c_void_p), ("pages_per_layer", C.c_longlong),
        ("last_token", C.c_void_p), ("dec_counters", C.c_void_p), ("dec_work", C.c_void_p),
        ("decode_impl", C.c_int),
        ("lora_R", C.c_int), ("lora_rank", C.c_int), ("lora_scale", C.c_float),
        ("lora", C.POINTER(MaceLoraLayer)),
        ("attn_pairs", C.c_int),
    ]


class MaceSavedActs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("x_in", "h1", "qkv", "o", "lse", "x_mid", "h2", "u", "a", "zm_o", "zm_d")]


class MaceTickBuffers(C.Structure):
    _fields_ = [
        *[(n, C.c_void_p) for n in ("x", "h", "qkv", "o", "lse", "hn", "u", "a")],
        ("sav", C.POINTER(MaceSavedActs)),
        *[(n, C.c_void_p) for n in ("rx", "rx2", "x_lmin", "rlse", "rh", "rqkv", "ro", "ru", "ra", "dx", "dy16", "df")],
        ("ld_df", C.c_int),
        *[(n, C.c_void_p) for n in ("da16", "du16", "do16", "dqkv", "dqkv16", "Dbuf", "ft_h", "ft_logits", "dlogits")],
        ("ld_vocab", C.c_int),
        *[(n, C.c_void_p) for n in ("dh", "row_lse", "row_lp", "dec_h", "dec_logits", "dec_tok", "dec_ws")],
        ("dec_ws_bytes", C.c_size_t),
        *[(n, C.c_void_p) for n in ("lp", "ref_lp", "loss", "margin", "coef", "ws")],
        ("ws_bytes", C.c_size_t),
        ("ld_h", C.c_int),
        *[(n, C.c_void_p) for n in ("lz", "lzm", "ldz")],
        ("dq_order", C.c_void_p),
        ("dec_keys", C.c_void_p),
    ]


class MaceTickDesc(C.Structure):
    _fields_ = [
        *[(n, C.c_int) for n in ("T", "ft0", "n_dec", "R", "n_pairs", "need_ref")],
        *[(n, C.c_void_p) for n in ("tokens", "pos", "row_seq", "row_kvi", "seqs", "tc_items")],
        ("n_tc", C.c_int), ("n_tc_inference", C.c_int),
        ("dec_items", C.c_void_p), ("n_dec_items", C.c_int),
        ("dec_slots", C.c_void_p), ("dec_rows", C.c_void_p),
        ("ptab_slots", C.c_void_p), ("ptab_rows", C.c_void_p), ("n_ptab", C.c_int), ("ptab_cols", C.c_int),
        ("page_copies", C.c_void_p), ("n_copies", C.c_int),
        *[(n, C.c_void_p) for n in ("ft_local_rows", "ft_targets", "pair_rows", "row_ps", "ref_cached", "ft_seqs",
                                    "ft_tc_items")],
        ("n_ft_tc", C.c_int),
        ("ft_row_seq", C.c_void_p), ("bwd_items", C.c_void_p), ("n_bwd", C.c_int),
        ("attn_events", C.c_void_p),
        ("gemm_events", C.c_void_p), ("gemm_events_cap", C.c_int), ("gemm_flops", C.c_void_p),
        ("gemm_count", C.c_void_p),
        ("row_tenant", C.c_void_p),
    ]


# MaceSeq is 8 x int32 (see include/mace_b200.h); built as numpy/torch int32 [S, 8] arrays
SEQ_FIELDS = ("kind", "q_start", "q_len", "slot", "n_pv", "kv_len", "hole0", "hole_len")

_vp, _i, _f, _ip = C.c_void_p, C.c_int, C.c_float, C.c_void_p

# (name, argtypes) for every symbol include/mace_b200.h declares; checked by tests/test_abi.py
SIGNATURES: dict[str, tuple[type, list]] = {
    "mace_version": (C.c_int, []),
    "mace_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "mace_ctx_destroy": (C.c_int, [C.c_void_p]),
    "mace_last_error": (C.c_char_p, [C.c_void_p]),
    "mace_launch_count": (C.c_longlong, [C.c_void_p]),
    "mace_debug_host_prof": (C.c_int, [C.POINTER(C.c_double)]),
    "mace_host_alg1": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double,
                                 C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_void_p,
                                 C.c_void_p, C.c_void_p]),
    "mace_host_head_stats": (C.c_int, [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 11 + [C.c_int, C.c_double,
                                                                                         C.c_void_p, C.c_void_p]),
    "mace_gemm_bf16": (C.c_int, [C.c_void_p, C.POINTER(MaceGemmArgs), C.c_void_p]),
    "mace_embed": (C.c_int, [_vp, _ip, _ip, _ip, _vp, _vp, _i, _i, _vp, _vp]),
    "mace_norm": (C.c_int, [_vp, _vp, _i, _ip, _i, _i, _vp, _vp, _i, _f, _vp, _i, _vp, _vp]),
    "mace_rope_kv": (C.c_int, [_vp, _vp, _i, _i, _i, _i, _ip, _ip, _ip, _vp, _vp, _vp, _i,
                               C.POINTER(MaceKvLayout), _vp, _vp, _vp]),
    "mace_act": (C.c_int, [_vp, _vp, _i, _i, _i, _vp, _vp]),
    "mace_argmax": (C.c_int, [_vp, _vp, _i, _i, _i, _ip, _vp]),
    "mace_argmax_keys": (C.c_int, [_vp, _vp, _i, _ip, _vp]),
    "mace_attn_fwd": (C.c_int, [_vp, C.POINTER(MaceAttnArgs), _vp]),
    "mace_dpo_fused": (C.c_int, [_vp, _vp, _i, _i, _i, _ip, _ip, _i, _ip, _vp, _f, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _i, _vp]),
    "mace_lora_mask": (C.c_int, [_vp, _vp, _i, _ip, _i, _i, _i, _f, _vp, _i, _vp]),
    "mace_f32_to_bf16_2d": (C.c_int, [_vp, _vp, _i, _i, _i, _vp, _i, _vp]),
    "mace_lora_bt_scatter": (C.c_int, [_vp, _vp, _i, _i, _vp, _i, _i, _vp]),
    "mace_adamw_segments": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, C.c_longlong] + [C.c_double] * 5
                            + [_i, _i, _vp]),
    "mace_dpo_scalar": (C.c_int, [_vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp]),
    "mace_adamw_masked": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_longlong, _vp, _vp, _i, _f, _f, _f, _f, _f, _i, _vp]),
    "mace_adamw_masked2": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_longlong, _vp, _vp, _i] + [C.c_double] * 5
                           + [_i, _i, _vp]),
    "mace_norm_bwd": (C.c_int, [_vp, _vp, _i, _ip, _vp, _i, _i, _i, _vp, _i, _f, _vp, _i, _ip, _vp, _vp, _vp,
                                C.c_size_t, _vp]),
    "mace_colsum_bf16": (C.c_int, [_vp, _vp, _i, _i, _i, _vp, _vp, C.c_size_t, _vp]),
    "mace_act_bwd": (C.c_int, [_vp, _vp, _vp, _i, _i, _i, _vp, _vp]),
    "mace_rope_bwd": (C.c_int, [_vp, _vp, _i, _i, _i, _i, _ip, _vp, _vp, _vp]),
    "mace_f32_to_bf16": (C.c_int, [_vp, _vp, C.c_longlong, _vp, _vp]),
    "mace_bf16_to_f32": (C.c_int, [_vp, _vp, C.c_longlong, _vp, _vp]),
    "mace_attn_bwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _ip, _i, _i, _vp, _vp, _vp]),
    "mace_attn_bwd2": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _ip, _i, _i, _vp, _vp, _vp, _vp]),
    "mace_kv_decode_alloc": (C.c_int, [_vp, C.POINTER(MaceKvLayout), _ip, _i, _vp]),
    "mace_kv_status": (C.c_int, [_vp, C.POINTER(MaceKvLayout), _ip]),
    "mace_kv_trim": (C.c_int, [_vp, C.POINTER(MaceKvLayout), _ip, _ip, _i, _vp]),
    "mace_kv_release": (C.c_int, [_vp, C.POINTER(MaceKvLayout), _ip, _i, _vp]),
    "mace_kv_compact": (C.c_int, [_vp, C.POINTER(MaceKvLayout), _ip, _i, _i, _i, _i, C.c_longlong, _vp, _vp, _vp]),
    "mace_kv_page_copy": (C.c_int, [_vp, _ip, _i, _i, _i, C.c_longlong, _i, _vp, _vp, _vp]),
    "mace_kv_set_prompt_tables": (C.c_int, [_vp, C.POINTER(MaceKvLayout), _ip, _ip, _i, _i, _vp]),
    "mace_scatter_tokens": (C.c_int, [_vp, _ip, _ip, _i, _ip, _vp]),
    "mace_model_create": (C.c_int, [_vp, C.POINTER(MaceModelDesc), C.POINTER(C.c_void_p)]),
    "mace_model_destroy": (C.c_int, [_vp]),
    "mace_tick_run": (C.c_int, [_vp, C.POINTER(MaceTickBuffers), C.POINTER(MaceTickDesc), _vp]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load the in-tree library once; raise loudly if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise MaceError(
                    f"{LIB_PATH} is missing: run `python -m paper_2510_03283_b200.build` "
                    "(the CUDA path has no CPU fallback)"
                )
            L = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
        return _lib


class Ctx:
    """One mace_ctx (per engine / thread). Owns nothing but the handle."""

    def __init__(self, device: int = 0):
        self.L = lib()
        h = C.c_void_p()
        rc = self.L.mace_ctx_create(device, C.byref(h))
        if rc != 0:
            raise MaceError(f"mace_ctx_create(device={device}) failed with status {rc} (needs an sm_100 GPU)")
        self.h = h

    def check(self, rc: int, what: str) -> None:
        if rc != 0:
            msg = self.L.mace_last_error(self.h).decode(errors="replace")
            raise MaceError(f"{what} failed ({rc}): {msg}")

    @property
    def launches(self) -> int:
        return int(self.L.mace_launch_count(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.L.mace_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
