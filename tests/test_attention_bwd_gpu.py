"""Attention backward of the FT rows (dense causal sequences) vs torch autograd in fp32 on the same bf16 inputs:
the tcgen05 kernel (head_dim 64 / 128, 128-key blocks) and the CUDA-core kernel (head_dim 32)."""
import math

import pytest
import torch

from paper_2510_03283_b200 import ops
from paper_2510_03283_b200._lib import MaceKvLayout

pytestmark = pytest.mark.gpu


def _items(lens, Hkv, kblk):
    items = []
    for si, n in enumerate(lens):
        nkb = (n + kblk - 1) // kblk
        for h in range(Hkv):
            for kb in range(nkb):
                items.append([si, h, kb, nkb - kb])
    items.sort(key=lambda x: -x[3])
    return torch.tensor(items, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("hd,Hq,Hkv,lens", [
    (64, 4, 4, (300, 128, 77)),          # GPT-2-like MHA, ragged lengths, one exact block
    (64, 8, 2, (513, 40)),               # GQA group 4
    (128, 4, 1, (260, 129)),             # Llama-3-8B head_dim, group 4
    (32, 4, 4, (150, 33)),               # tiny: CUDA-core kernel
])
def test_attention_backward(ctx, hd, Hq, Hkv, lens):
    torch.manual_seed(hd + Hq + sum(lens))
    W = (Hq + 2 * Hkv) * hd
    T = sum(lens)
    qkv = (torch.randn(T, W, device="cuda") * 0.5).bfloat16()
    dout = torch.randn(T, Hq * hd, device="cuda").bfloat16()
    seqs, q0 = [], 0
    for n in lens:
        seqs.append([2, q0, n, -1, 0, n, -1, 0])
        q0 += n
    seqs_t = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    fwd_items = torch.tensor([[si, hq, qb, 0] for si, n in enumerate(lens) for hq in range(Hq)
                              for qb in range((n + 127) // 128)], dtype=torch.int32, device="cuda")
    o = torch.zeros(T, Hq * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros(T, Hq, device="cuda")
    lay = MaceKvLayout(ptab=None, max_prompt_pages=0, dtab=None, max_dec_pages=0, dec_base=None, dec_first=None,
                       dec_end=None, free_stack=None, free_top=None, stack_cap=0, n_kv_heads=Hkv)
    ops.attn_fwd(ctx, qkv, Hq, Hkv, hd, seqs_t, fwd_items, None, lay, None, None, o, lse=lse)
    dqkv = ops.attn_bwd(ctx, qkv, o, dout, lse, Hq, Hkv, hd, seqs_t, _items(lens, Hkv, 128 if hd >= 64 else 64))
    torch.cuda.synchronize()
    # reference: fp32 autograd of causal softmax attention per sequence / head
    G = Hq // Hkv
    x = qkv.float().requires_grad_(True)
    outs = []
    q0 = 0
    for n in lens:
        blk = x[q0: q0 + n]
        q = blk[:, : Hq * hd].view(n, Hq, hd).transpose(0, 1)
        k = blk[:, Hq * hd: (Hq + Hkv) * hd].view(n, Hkv, hd).transpose(0, 1).repeat_interleave(G, 0)
        v = blk[:, (Hq + Hkv) * hd:].view(n, Hkv, hd).transpose(0, 1).repeat_interleave(G, 0)
        s = q @ k.transpose(1, 2) / math.sqrt(hd)
        s = s.masked_fill(torch.ones(n, n, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
        outs.append((torch.softmax(s, -1) @ v).transpose(0, 1).reshape(n, Hq * hd))
        q0 += n
    torch.cat(outs).backward(dout.float())
    ref = x.grad
    err = (dqkv - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 2e-2 * scale + 1e-3, f"max err {err} vs max |grad| {scale}"
    rel = ((dqkv - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel
