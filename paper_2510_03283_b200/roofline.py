"""Whole-tick roofline of the hybrid iteration (roofline time = Σ_kernels max(F_k / F_peak, B_k / B_peak)).

Algorithmic work of one tick from its row tables (TickBatch) and the model shapes -- what the tick must do, not what
the kernels happen to move:

  tensor FLOPs  every projection / lm_head GEMM of the tick (measured exactly by the tick executor's GEMM events:
                2·M·N·K per launch, forward, FT sub-passes and backward) plus the tensor-core attention: 4·hd·Hq per
                visible causal (query, key) pair for prefill / FT sequences in every layer they run through, the FT
                sub-passes (pi_ref and policy) through the selected layers, and 2.5x that (S and dP recomputed,
                dV, dK, dQ) for the FT backward of the selected layers;
  HBM bytes     paged decode attention (every visible K / V row once + q / o rows; measured per launch from the
                device tables), and the row kernels: embedding, the two norms and RoPE / KV scatter of every layer
                pass, the decode head (norm; its argmax is fused into the lm_head GEMM), the DPO logit passes, the FT backward's row kernels
                and the masked AdamW (30 B per updated parameter).

roofline_ms = tensor_flops / tensor_peak + hbm_bytes / hbm_peak (each class is bound by one resource).
"""
from __future__ import annotations

import numpy as np

from .batch import KIND_FT, KIND_PREFILL


def causal_pairs(seqs: np.ndarray) -> tuple[int, int]:
    """(prefill pairs, FT pairs): visible (query, key) pairs of the tick's tensor-core attention sequences."""
    pre = ft = 0
    for kind, _, q, _, _, kv, h0, hl in seqs.tolist():
        if kind == KIND_PREFILL:
            pre += q * (kv - q) + q * (q + 1) // 2
        elif kind == KIND_FT:
            n = q
            lost = max(0, n - (h0 + hl)) * hl if hl > 0 else 0
            ft += n * (n + 1) // 2 - lost
    return pre, ft


def tick_extras(batch, cfg, n_sel: int, n_updated_params: int, lora: bool = False) -> dict:
    """Attention FLOPs and row-kernel bytes of one tick (the GEMM FLOPs and decode-attention bytes are measured)."""
    L, D, hd, Hq, Hkv = cfg.n_layers, cfg.d_model, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    V, F, UP, QKV = cfg.vocab, cfg.ffn, cfg.up_dim, cfg.qkv_dim
    T, ft0 = batch.T, batch.ft0
    n_ft = T - ft0
    has_ft = n_ft > 0 and len(batch.ft_pairs) > 0
    R = int(batch.ft_logit_rows.shape[0])
    n_dec = batch.n_dec
    l_min = L - n_sel
    pre_pairs, ft_pairs = causal_pairs(batch.seqs)
    att = 4 * hd * Hq
    # forward attention: prefill sequences through every layer; FT sequences through the shared layers below l_min
    # (or all layers when the tick has no FT step), then twice (pi_ref, policy) through the selected layers
    shared_ft_layers = l_min if has_ft else L
    flops = att * (pre_pairs * L + ft_pairs * shared_ft_layers)
    if has_ft:
        flops += att * ft_pairs * n_sel * 2 + 2.5 * att * ft_pairs * n_sel
    # row-kernel bytes
    row = lambda n, per: n * per  # noqa: E731
    norm_b = D * (4 + 2)
    rope_b = QKV * 2 + (Hq + Hkv) * hd * 2 + 2 * Hkv * hd * 2
    layer_rows = (T * l_min + ft0 * n_sel) if has_ft else T * L
    byts = row(T, D * (2 + 4))                                   # embedding
    byts += layer_rows * (2 * norm_b + rope_b)
    byts += row(n_dec, norm_b + 8)                               # decode head: norm + argmax key (fused lm_head)
    if has_ft:
        sub_rows = 2 * n_sel * n_ft                              # pi_ref + policy sub-passes
        byts += sub_rows * (2 * norm_b + QKV * 2 * 2 + UP * 2 + F * 2 + 2 * 4 * D)  # + unfused act, saved copies
        byts += 2 * row(R, norm_b + V * 4 * 2) + row(R, V * 2)   # lm_head logits of both passes, DPO reads, dlogits
        bwd_per_row = 2 * (D * 4 * 3) + UP * 2 * 2 + F * 2 * 2 + QKV * 4 * 3 + Hq * hd * 2 * 2
        byts += n_sel * n_ft * bwd_per_row                       # norm / act / rope backward, conversions
        byts += 30 * n_updated_params                            # masked AdamW
    return {"attn_flops": float(flops), "row_bytes": float(byts)}
