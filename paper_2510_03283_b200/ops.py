"""Thin torch-tensor front end over the C-ABI (device pointers + the current CUDA stream).

torch is plumbing here (device memory, streams); every op below is one or more launches of the
hand-written sm_100a kernels in csrc/. Shapes are validated on the host before the launch.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import Ctx, MaceGemmArgs

EPI = {"bf16": 0, "f32": 1, "f32_add": 2, "f32_atomic": 3, "bf16_gelu": 4, "bf16_swiglu": 5, "argmax": 6}


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def gemm(
    ctx: Ctx,
    a: torch.Tensor,
    b: torch.Tensor,
    out: torch.Tensor | None = None,
    *,
    mode: str = "bf16",
    bias: torch.Tensor | None = None,
    a_mn: bool = False,
    b_mn: bool = False,
    alpha: float = 1.0,
    split_k: int = 0,
    workspace: torch.Tensor | None = None,
    stream: torch.cuda.Stream | None = None,
    b_static: bool = False,
) -> torch.Tensor:
    """out[M,N] (op)= alpha * A[M,K] . B[N,K]^T.

    ``a`` is [M,K] (K-major) or, with ``a_mn``, [K,M]; ``b`` is [N,K] or, with ``b_mn``, [K,N].
    Leading dims may be padded (row stride used as ld) but the inner dim must be contiguous.
    """
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    assert a.stride(1) == 1 and b.stride(1) == 1
    if a_mn:
        K, M = a.shape
    else:
        M, K = a.shape
    if b_mn:
        Kb, N = b.shape
    else:
        N, Kb = b.shape
    assert Kb == K, f"K mismatch {K} vs {Kb}"
    if mode == "bf16_swiglu":  # b = [gate; up] stacked: 2N rows, N outputs
        assert N % 2 == 0 and not b_mn
        N //= 2
    if mode == "argmax":  # out: int64 keys [M], zeroed (see argmax_keys)
        if out is None:
            out = torch.zeros(M, device=a.device, dtype=torch.int64)
        assert out.dtype == torch.int64 and out.numel() >= M and out.is_contiguous()
    else:
        if out is None:
            assert mode in ("bf16", "f32", "bf16_gelu", "bf16_swiglu")
            out = torch.empty(M, N, device=a.device, dtype=torch.float32 if mode == "f32" else torch.bfloat16)
        assert out.shape[0] >= M and out.shape[1] >= N and out.stride(1) == 1
        assert out.dtype == (torch.bfloat16 if mode in ("bf16", "bf16_gelu", "bf16_swiglu") else torch.float32)
    if bias is not None:
        assert bias.dtype == torch.bfloat16 and bias.numel() == N
    g = MaceGemmArgs(
        a=_ptr(a), lda=a.stride(0), a_mn_major=int(a_mn),
        b=_ptr(b), ldb=b.stride(0), b_mn_major=int(b_mn),
        M=M, N=N, K=K,
        out=_ptr(out), ldo=0 if mode == "argmax" else out.stride(0), mode=EPI[mode],
        bias=_ptr(bias), alpha=float(alpha), split_k=int(split_k),
        workspace=_ptr(workspace), workspace_bytes=0 if workspace is None else workspace.numel() * workspace.element_size(),
        flags=1 if b_static else 0,
    )
    ctx.check(ctx.L.mace_gemm_bf16(ctx.h, C.byref(g), _stream(stream)), "mace_gemm_bf16")
    return out


def argmax_keys(ctx: Ctx, keys: torch.Tensor, n: int | None = None, out: torch.Tensor | None = None,
                stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Token ids from the keys of an ``argmax`` GEMM (first index on ties); resets the keys to zero."""
    n = keys.numel() if n is None else n
    assert keys.dtype == torch.int64 and keys.is_contiguous()
    if out is None:
        out = torch.empty(n, device=keys.device, dtype=torch.int32)
    ctx.check(ctx.L.mace_argmax_keys(ctx.h, _ptr(keys), n, _ptr(out), _stream(stream)), "mace_argmax_keys")
    return out


def attn_fwd(
    ctx: Ctx,
    qkv: torch.Tensor,
    Hq: int,
    Hkv: int,
    hd: int,
    seqs: torch.Tensor,
    tc_items: torch.Tensor | None,
    dec_items: torch.Tensor | None,
    kv_layout,
    k_pool: torch.Tensor | None,
    v_pool: torch.Tensor | None,
    out: torch.Tensor,
    lse: torch.Tensor | None = None,
    head_norm: torch.Tensor | None = None,
    stream: torch.cuda.Stream | None = None,
    dec_workspace: torch.Tensor | None = None,
    dec_counters: torch.Tensor | None = None,
    dec_work: torch.Tensor | None = None,
    decode_impl: int = 0,
    tc_pairs: bool = False,
) -> torch.Tensor:
    """Ragged paged attention of one tick (prefill + FT tiles on tcgen05, decode rows streamed)."""
    from ._lib import MaceAttnArgs

    T = qkv.shape[0]
    assert qkv.dtype == torch.bfloat16 and qkv.shape[1] == (Hq + 2 * Hkv) * hd and qkv.is_contiguous()
    assert seqs.dtype == torch.int32 and seqs.shape[1] == 8
    a = MaceAttnArgs(
        qkv=qkv.data_ptr(), T=T, Hq=Hq, Hkv=Hkv, hd=hd, seqs=seqs.data_ptr(),
        tc_items=_ptr(tc_items), n_tc=0 if tc_items is None else tc_items.shape[0],
        dec_items=_ptr(dec_items), n_dec=0 if dec_items is None else dec_items.shape[0],
        kv=kv_layout,
        k_pool=_ptr(k_pool), v_pool=_ptr(v_pool), pool_pages=0 if k_pool is None else k_pool.shape[0],
        out=out.data_ptr(), lse=_ptr(lse), head_norm=_ptr(head_norm), scale=0.0,
        dec_workspace=_ptr(dec_workspace),
        dec_workspace_bytes=0 if dec_workspace is None else dec_workspace.numel() * dec_workspace.element_size(),
        dec_counters=_ptr(dec_counters), dec_work=_ptr(dec_work), decode_impl=int(decode_impl), tc_pairs=int(tc_pairs),
    )
    ctx.check(ctx.L.mace_attn_fwd(ctx.h, C.byref(a), _stream(stream)), "mace_attn_fwd")
    return out


def attn_bwd(
    ctx: Ctx,
    qkv: torch.Tensor,
    o: torch.Tensor,
    dout: torch.Tensor,
    lse: torch.Tensor,
    Hq: int,
    Hkv: int,
    hd: int,
    seqs: torch.Tensor,
    items: torch.Tensor,
    dqkv: torch.Tensor | None = None,
    stream: torch.cuda.Stream | None = None,
    ordered: bool = True,
) -> torch.Tensor:
    """Attention backward of dense causal sequences: dqkv fp32 [T, (Hq+2Hkv)*hd] (dQ, dK, dV in the qkv layout).
    ordered: deterministic dQ accumulation (mace_attn_bwd2) instead of fp32 atomics.
    ``items`` int32 [n, 4] = (seq, kv_head, key_block, steps) with 128-key blocks (hd 64/128) or 64 (hd 32)."""
    T = qkv.shape[0]
    if dqkv is None:
        dqkv = torch.zeros(T, qkv.shape[1], dtype=torch.float32, device=qkv.device)
    Dbuf = torch.empty(T, Hq, dtype=torch.float32, device=qkv.device)
    order = torch.zeros(T * Hq, dtype=torch.int32, device=qkv.device) if ordered else None
    ctx.check(ctx.L.mace_attn_bwd2(ctx.h, _ptr(qkv), _ptr(o), _ptr(dout), _ptr(lse), T, Hq, Hkv, hd, _ptr(seqs),
                                   _ptr(items), items.shape[0], 0, _ptr(Dbuf), _ptr(dqkv), _ptr(order),
                                   _stream(stream)), "attn_bwd")
    if ordered:  # every counter is left at zero by its last contributor
        assert int(order.abs().sum()) == 0
    return dqkv
