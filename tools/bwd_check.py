"""Per-kernel precision of the fine-tune backward at Llama-3-8B (C4) shapes against fp32 torch on the same bf16
inputs: every GEMM layout tick.cu's layer_bwd / ft_step issue, the hd-128 GQA attention backward over C4-long
fine-tune sequences, and the RMSNorm backward. Prints rel-L2 per op (run on the B200)."""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx, MaceKvLayout  # noqa: E402
from paper_2510_03283_b200.build import build  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False


def rel(a, b):
    return float((a.float() - b.float()).norm() / (b.float().norm() + 1e-30))


def main():
    build()
    ctx = Ctx(0)
    dev = "cuda"
    n, R, D, F, V = int(sys.argv[1]) if len(sys.argv) > 1 else 5200, 130, 4096, 14336, 128256
    Hq, Hkv, hd = 32, 8, 128
    HO, QKV, UP = Hq * hd, (Hq + 2 * Hkv) * hd, 2 * F
    g = torch.Generator(device=dev).manual_seed(0)
    rnd = lambda *s, sc=1.0: (torch.randn(*s, device=dev, generator=g) * sc).bfloat16()  # noqa: E731
    ws = torch.empty(16 << 20, device=dev)
    # (name, A, a_mn, B, b_mn): out = A . B^T with A [M,K] (or [K,M] MN-major), B [N,K] (or [K,N])
    vp = (V + 7) // 8 * 8
    dl = torch.zeros(R, vp, device=dev, dtype=torch.bfloat16)
    dl[:, :V] = rnd(R, V, sc=1e-3)
    E = rnd(V, D, sc=0.1)
    cases = [
        ("dh = dlogits . E       (M=R, K=V)", dl[:, :V], False, E, True),
        ("dW_down = dy^T a        (K=n)", rnd(n, D), True, rnd(n, F), True),
        ("da = dy . W_down        (K=D)", rnd(n, D), False, rnd(D, F, sc=0.02), True),
        ("dW_up = du^T h2         (K=n)", rnd(n, UP), True, rnd(n, D), True),
        ("df = du . W_up          (K=UP)", rnd(n, UP), False, rnd(UP, D, sc=0.02), True),
        ("dW_o = dy^T o           (K=n)", rnd(n, D), True, rnd(n, HO), True),
        ("do = dy . W_o           (K=D)", rnd(n, D), False, rnd(D, HO, sc=0.02), True),
        ("dW_qkv = dqkv^T h1      (K=n)", rnd(n, QKV), True, rnd(n, D), True),
        ("df = dqkv . W_qkv       (K=QKV)", rnd(n, QKV), False, rnd(QKV, D, sc=0.02), True),
    ]
    for name, A, a_mn, B, b_mn in cases:
        out = ops.gemm(ctx, A, B, mode="f32", a_mn=a_mn, b_mn=b_mn, workspace=ws)
        Af = (A.t() if a_mn else A).float()
        Bf = (B.t() if b_mn else B).float()
        ref = Af @ Bf.t()
        acc0 = torch.randn_like(ref)
        acc = acc0.clone()
        ops.gemm(ctx, A, B, acc, mode="f32_add", a_mn=a_mn, b_mn=b_mn, workspace=ws)
        torch.cuda.synchronize()
        print(f"gemm {name}: out {tuple(ref.shape)} rel-L2 f32 {rel(out, ref):.2e}  f32_add {rel(acc - acc0, ref):.2e}")
    # attention backward, C4-long fine-tune sequences (GQA 32/8, hd 128)
    lens = [1310, 1340, 1200, 1290]
    T = sum(lens)
    W = QKV
    qkv = rnd(T, W, sc=0.5)
    dout = rnd(T, HO)
    seqs, q0 = [], 0
    for L in lens:
        seqs.append([2, q0, L, -1, 0, L, -1, 0])
        q0 += L
    seqs_t = torch.tensor(seqs, dtype=torch.int32, device=dev)
    fwd_items = torch.tensor([[si, hq, qb, 0] for si, L in enumerate(lens) for hq in range(Hq)
                              for qb in range((L + 127) // 128)], dtype=torch.int32, device=dev)
    o = torch.zeros(T, HO, dtype=torch.bfloat16, device=dev)
    lse = torch.zeros(T, Hq, device=dev)
    lay = MaceKvLayout(n_kv_heads=Hkv)
    ops.attn_fwd(ctx, qkv, Hq, Hkv, hd, seqs_t, fwd_items, None, lay, None, None, o, lse=lse)
    items = []
    for si, L in enumerate(lens):
        nkb = (L + 127) // 128
        for h in range(Hkv):
            for kb in range(nkb):
                items.append([si, h, kb, nkb - kb])
    items.sort(key=lambda x: -x[3])
    dqkv = ops.attn_bwd(ctx, qkv, o, dout, lse, Hq, Hkv, hd, seqs_t, torch.tensor(items, dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    G = Hq // Hkv
    x = qkv.float().requires_grad_(True)
    outs, q0 = [], 0
    for L in lens:
        blk = x[q0: q0 + L]
        q = blk[:, :HO].view(L, Hq, hd).transpose(0, 1)
        k = blk[:, HO: HO + Hkv * hd].view(L, Hkv, hd).transpose(0, 1).repeat_interleave(G, 0)
        v = blk[:, HO + Hkv * hd:].view(L, Hkv, hd).transpose(0, 1).repeat_interleave(G, 0)
        s = q @ k.transpose(1, 2) / math.sqrt(hd)
        s = s.masked_fill(torch.ones(L, L, device=dev, dtype=torch.bool).triu(1), float("-inf"))
        outs.append((torch.softmax(s, -1) @ v).transpose(0, 1).reshape(L, HO))
        q0 += L
    ref_o = torch.cat(outs)
    ref_o.backward(dout.float())
    print(f"attn fwd hd128 GQA: rel-L2 o {rel(o, ref_o):.2e}")
    for nm, sl in (("dq", slice(0, HO)), ("dk", slice(HO, HO + Hkv * hd)), ("dv", slice(HO + Hkv * hd, W))):
        print(f"attn bwd hd128 GQA {nm}: rel-L2 {rel(dqkv[:, sl], x.grad[:, sl]):.2e}")
    # RMSNorm backward at d 4096 over n rows
    xs = torch.randn(n, D, device=dev)
    w = (1 + 0.05 * torch.randn(D, device=dev)).bfloat16()
    dy = torch.randn(n, D, device=dev)
    dx = torch.randn(n, D, device=dev)
    dx0 = dx.clone()
    dw = torch.zeros(D, device=dev)
    ctx.check(ctx.L.mace_norm_bwd(ctx.h, xs.data_ptr(), D, None, dy.data_ptr(), D, n, D, w.data_ptr(), 0, 1e-5,
                                  dx.data_ptr(), D, None, dw.data_ptr(), None, ws.data_ptr(), ws.numel() * 4, None),
              "norm_bwd")
    torch.cuda.synchronize()
    xr = xs.clone().requires_grad_(True)
    wr = w.float().requires_grad_(True)
    y = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * wr
    y.backward(dy)
    print(f"rmsnorm bwd d4096: rel-L2 dx {rel(dx - dx0, xr.grad):.2e}  dw {rel(dw, wr.grad):.2e}")


if __name__ == "__main__":
    main()
