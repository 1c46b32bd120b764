"""The fine-tune kernels against the reference and exact restatements (B200, through the C-ABI).

* DPO scalar stage (csrc/dpo_adamw.cu dpo_scalar, shared by mace_dpo_fused's pair stage) on the reference's
  own golden vectors (tests/golden/dpo_golden.json, generated from macesim.alignment.dpo_loss):
  relative error <= 1e-6 required; the fp64 device stage is in fact within a few ulp.
* mace_dpo_fused end to end: per-pair loss = macesim dpo_loss of the kernel's own log-prob sums (<= 1e-6
  relative after the fp32 store), log-probs vs an fp64 log-softmax, dlogits vs coef * (onehot - softmax).
* masked AdamW (scalar and float4 kernels): BIT-EXACT against a numpy fp32 restatement with the kernel's
  operation order, over 5 steps and many segments, and within 8 fp32 ulp of torch.optim.AdamW itself (torch's
  CPU kernels may fuse multiply-adds, so bit equality with torch is not defined); the bf16 working copies
  equal bf16(master) everywhere and are untouched outside the selected segments.
"""
import ctypes as C
import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

from parity_util import adamw_np

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden" / "dpo_golden.json"


def _p(t):
    return C.c_void_p(t.data_ptr())


def test_dpo_scalar_stage_on_reference_golden(ctx):
    g = json.loads(GOLD.read_text())
    rows = g["known"] + g["samples"]
    m = torch.tensor([r["m"] for r in rows], dtype=torch.float64, device="cuda")
    b = torch.tensor([r["beta"] for r in rows], dtype=torch.float64, device="cuda")
    zero = torch.zeros_like(m)
    loss, marg, sig = torch.empty_like(m), torch.empty_like(m), torch.empty_like(m)
    ctx.check(ctx.L.mace_dpo_scalar(ctx.h, _p(m), _p(zero), _p(b), len(rows), _p(loss), _p(marg), _p(sig), None),
              "dpo_scalar")
    torch.cuda.synchronize()
    loss, marg, sig = loss.cpu().tolist(), marg.cpu().tolist(), sig.cpu().tolist()
    worst = 0.0
    for r, l, mm, sg in zip(rows, loss, marg, sig):
        assert mm == r["m"]
        rel = abs(l - r["ref"]) / abs(r["ref"])
        worst = max(worst, rel)
        assert rel <= 1e-6, (r, l)
        if "f128" in r:
            assert abs(l - r["f128"]) <= 1e-9 * max(1.0, abs(r["f128"]))  # A1 tolerance, test_acceptance.py:47-54
        if "want" in r:
            assert abs(l - r["want"]) < 1e-12
        if "want_below" in r:
            assert l < r["want_below"]
        x = -r["beta"] * r["m"]
        assert abs(sg - 1.0 / (1.0 + math.exp(-x))) <= 1e-12
    print(f"dpo scalar stage: worst relative error vs macesim.dpo_loss {worst:.2e} over {len(rows)} vectors")


def test_dpo_fused_matches_reference_scalar_stage(ctx):
    from macesim.alignment import MarginSample, dpo_loss

    torch.manual_seed(3)
    V, ld, beta = 50257, 50264, 0.7
    lens = [(37, 41), (5, 9), (120, 64)]
    P = len(lens)
    pair_rows, row_ps, r0 = [], [], 0
    for p, (nc, nr) in enumerate(lens):
        pair_rows.append([r0, nc, r0 + nc, nr])
        row_ps += [2 * p] * nc + [2 * p + 1] * nr
        r0 += nc + nr
    R = r0
    logits = torch.zeros(R, ld, dtype=torch.float32, device="cuda")
    logits[:, :V] = torch.randn(R, V, device="cuda") * 3.0
    tg = torch.randint(0, V, (R,), dtype=torch.int32, device="cuda")
    pr = torch.tensor(pair_rows, dtype=torch.int32, device="cuda")
    ps = torch.tensor(row_ps, dtype=torch.int32, device="cuda")
    ref = (torch.randn(P, 2, device="cuda") * 40.0 - 400.0).float()
    f32 = lambda *s: torch.empty(*s, dtype=torch.float32, device="cuda")  # noqa: E731
    row_lse, row_lp, lp, loss, margin, coef = f32(R), f32(R), f32(P, 2), f32(P), f32(P), f32(P, 2)
    dl = torch.empty(R, ld, dtype=torch.bfloat16, device="cuda")
    ctx.check(ctx.L.mace_dpo_fused(ctx.h, _p(logits), R, V, ld, _p(tg), _p(pr), P, _p(ps), _p(ref), C.c_float(beta),
                                   _p(row_lse), _p(row_lp), _p(lp), _p(loss), _p(margin), _p(coef), _p(dl), ld, None),
              "dpo_fused")
    torch.cuda.synchronize()
    lg = logits[:, :V].double().cpu()
    want_lp_rows = torch.log_softmax(lg, -1).gather(1, tg.long().cpu()[:, None])[:, 0]
    assert torch.allclose(row_lp.double().cpu(), want_lp_rows, rtol=1e-5, atol=2e-5)
    lp_h, ref_h = lp.cpu().double(), ref.cpu().double()
    for p, (c0, nc, j0, nr) in enumerate(pair_rows):
        assert abs(lp_h[p, 0].item() - want_lp_rows[c0:c0 + nc].sum().item()) <= 1e-5 * nc * 20
        want = dpo_loss(MarginSample(lp_h[p, 0].item() - ref_h[p, 0].item(), lp_h[p, 1].item() - ref_h[p, 1].item()), beta)
        got = loss[p].item()
        assert abs(got - want) <= 1e-6 * abs(want) + 1e-30, (p, got, want)
        m = (lp_h[p, 0] - ref_h[p, 0]) - (lp_h[p, 1] - ref_h[p, 1])
        assert margin[p].item() == np.float32(m.item())
        sg = 1.0 / (1.0 + math.exp(beta * m.item()))
        assert abs(coef[p, 0].item() + beta * sg / P) <= 1e-6 * beta * sg / P + 1e-30
    # dlogits = coef[row] * (onehot - softmax): bf16 storage
    sm = torch.softmax(lg, -1)
    oh = torch.zeros_like(sm)
    oh[torch.arange(R), tg.long().cpu()] = 1.0
    cr = coef.cpu().double().reshape(-1)[torch.tensor(row_ps)]
    want_dl = cr[:, None] * (oh - sm)
    got_dl = dl[:, :V].double().cpu()
    assert ((got_dl - want_dl).abs() <= 2 ** -8 * want_dl.abs() + 1e-12).all()


@pytest.mark.parametrize("sizes,vec4", [((768, 768, 2304 * 64, 2304, 3072 * 33, 13), False),
                                        ((768, 768, 2304 * 64, 2304, 3072 * 33, 4096 * 7), True)])
def test_masked_adamw_bit_exact(ctx, sizes, vec4):
    torch.manual_seed(1)
    n = sum(sizes)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    # bf16 working copies live inside a larger weight buffer: only the selected segments may change
    starts = [int(o) + 8 * i for i, o in enumerate(offs[:-1])]  # distinct 16-byte aligned bf16 copies
    pool = torch.randn(starts[-1] + sizes[-1] + 64, dtype=torch.bfloat16, device="cuda")
    pool_before = pool.clone()
    master = torch.cat([pool[s: s + k].float() for s, k in zip(starts, sizes)])
    m, v = torch.zeros_like(master), torch.zeros_like(master)
    seg_off = torch.from_numpy(offs).cuda()
    seg_ptr = torch.tensor([pool.data_ptr() + 2 * s for s in starts], dtype=torch.int64, device="cuda")
    hp = (1e-3, 0.9, 0.999, 1e-8, 0.01)
    P, M, Vv = master.cpu().numpy().copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    for step in range(1, 6):
        g = torch.randn(n, device="cuda") * torch.logspace(-6, 0, n, device="cuda")
        ctx.check(ctx.L.mace_adamw_masked2(ctx.h, _p(master), _p(m), _p(v), _p(g), n, _p(seg_off), _p(seg_ptr),
                                           len(sizes), *map(C.c_double, hp), step, int(vec4), None), "adamw")
        gh = g.cpu().numpy()
        P_prev, M_prev, V_prev = P, M, Vv
        P, M, Vv = adamw_np(P, M, Vv, gh, *hp, step)
        torch.cuda.synchronize()
        assert np.array_equal(master.cpu().numpy().view(np.int32), P.view(np.int32)), f"master, step {step}"
        assert np.array_equal(m.cpu().numpy().view(np.int32), M.view(np.int32)), f"m, step {step}"
        assert np.array_equal(v.cpu().numpy().view(np.int32), Vv.view(np.int32)), f"v, step {step}"
        # torch.optim.AdamW taking the same step from the same state: within 4 ulp of the larger of the weight and
        # the step size. torch's CPU kernels may contract lerp / addcmul into FMAs (CPU-dependent vectorisation) and
        # addcdiv rounds (value*m)/denom where the kernel rounds value*(m/denom): ulp-level differences per step
        tp = torch.nn.Parameter(torch.from_numpy(P_prev.copy()))
        opt = torch.optim.AdamW([tp], lr=hp[0], betas=(hp[1], hp[2]), eps=hp[3], weight_decay=hp[4], foreach=False)
        opt.state[tp] = {"step": torch.tensor(float(step - 1)), "exp_avg": torch.from_numpy(M_prev.copy()),
                         "exp_avg_sq": torch.from_numpy(V_prev.copy())}
        tp.grad = g.cpu().clone()
        opt.step()
        scale = np.maximum(np.maximum(np.abs(tp.detach().numpy()), np.abs(P_prev)), np.float32(hp[0]))
        err = np.abs(P - tp.detach().numpy()) / np.spacing(scale)
        assert err.max() <= 4, f"torch AdamW, step {step}: {err.max()} ulp at {int(err.argmax())}"
    mask = torch.zeros(pool.numel(), dtype=torch.bool, device="cuda")
    for s, k, o in zip(starts, sizes, offs[:-1]):
        assert torch.equal(pool[s: s + k], master[o: o + k].to(torch.bfloat16))
        mask[s: s + k] = True
    assert torch.equal(pool[~mask], pool_before[~mask]), "AdamW wrote outside the selected segments"
