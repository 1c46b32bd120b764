"""Shared checker for the tick-replay parity tests (C1, the model families, the full-shape samples).

Every tick GpuEngine executed on the B200 is replayed by TWO restatements from the same recorded tick batch:
the fp32 oracle (oracle/model_ref.py:TickOracle) and the same oracle with bf16 rounding at the points where the
device stores bf16 (Bf16EmulationModel: an independent torch implementation of the same numerics class). The
latter's distance to fp32 is the noise floor of bf16 arithmetic for that tick; SURVEY.md §8(c)'s absolute bounds
are asserted where they sit above that floor and reported (stats) everywhere:

  decode logits      rel-L2(gpu, f32) <= max(1e-2, 1.5 * rel-L2(bf16 emulation, f32)) per tick
  decode token ids   bit-exact, except oracle near-ties (top-1/top-2 gap < 0.05): counted, <= 5% of tokens
  DPO margin / loss  EXACT (m = 0, L = ln 2) while pi_theta == pi_ref (a pair's first step: same kernels, rows);
                     otherwise, over all n later-step pairs: rms(gpu - f32) <= r * rms(bf16 emulation - f32) + 1e-3,
                     r = max(1.5, sqrt(F_0.995(n, n))) (the rms ratio of two equal-variance noise samples of n pairs,
                     n >= 20); every pair |m - m_f32| <= max(0.5 nat, 2 x the emulation's worst) and
                     |L - L_f32| <= beta * |m - m_f32|.
                     (A margin is a difference of two log-prob sums of hundreds of nats computed under weights a
                     few bf16 ulps apart; its bf16 rounding noise, ~0.05-0.5 nat, is far above §8(c)'s 1e-2 and is
                     shown by the independent emulation as much as by the device.)
  selected grads     taken by both restatements AT THE DEVICE'S MARGINS (the DPO outer derivative
                     -beta*sigma(-beta*m) is a function of the margin, whose forward noise is checked above), so
                     the comparison measures the backward alone; rel-L2 per (tick, tensor), over all of them:
                     rms(gpu) <= 1.5 * rms(bf16 emulation) + 2e-3 and worst(gpu) <= max(2 * worst(bf16
                     emulation), 0.02)
  AdamW (in situ)    the device masters / m / v after each update are BIT-EXACT with the numpy fp32
                     restatement of the kernel (adamw_np) applied to the device's own pre-update state and
                     gradient
  updated weights    elementwise §8(c) bound |dw - dw_f32| <= 1e-2 * max|dw_f32| + 1 fp32 ulp(w) from the same
                     pre-update state; the mean (over updates) fraction of elements outside it must not exceed the
                     bf16 emulation's own * 1.5 + 1e-3 (Adam's sign-like step turns every gradient sign flip near
                     zero into a 2*lr move, for any bf16 implementation)
"""
from __future__ import annotations

import math

import numpy as np
import torch
from scipy.stats import f as f_dist


def adamw_np(p, m, v, g, lr, b1, b2, eps, wd, step):
    """numpy fp32 restatement of csrc/dpo_adamw.cu adamw_elem (per-op IEEE rounding, the kernel's order); the
    scalars are derived exactly as mace_adamw_masked2 derives them from its double arguments."""
    f = np.float32
    bc1, bc2 = 1.0 - b1 ** step, 1.0 - b2 ** step
    decay, w1, w2 = f(1.0 - lr * wd), f(1.0 - b1), f(1.0 - b2)
    ss, sb = f(lr / bc1), f(math.sqrt(bc2))
    p = p * decay
    m = m + w1 * (g - m)
    v = v * f(b2) + w2 * (g * g)
    denom = np.sqrt(v) / sb + f(eps)
    p = p - ss * (m / denom)
    return p, m, v


def _rel(a, b) -> float:
    return float((a.float() - b.float()).norm() / (b.float().norm() + 1e-30))


def adamw_np_tenants(pre, g, tenants, steps, widths, rank, tcfg):
    """LoRA: the per-tenant AdamW restatement over the flat buffers -- for each stepping tenant u (with its own
    step count steps[u]) the rows [u * rank, (u + 1) * rank) of every adapter tensor [R, width] (flat order);
    every other element stays as it was."""
    out = [a.copy() for a in pre]
    for u in tenants:
        idx, off = [], 0
        for wd, numel in widths:
            idx.append(np.arange(off + u * rank * wd, off + (u + 1) * rank * wd))
            off += numel
        idx = np.concatenate(idx)
        res = adamw_np(pre[0][idx], pre[1][idx], pre[2][idx], g[idx], tcfg.lr, tcfg.beta1, tcfg.beta2, tcfg.eps,
                       tcfg.weight_decay, int(steps[u]))
        for a, r in zip(out, res):
            a[idx] = r
    return tuple(out)


def check_records(eng, w, cfg, tcfg, device="cpu", max_tie_frac=0.05, label=""):
    from oracle.model_ref import TickOracle
    from paper_2510_03283_b200.config import trainable_param_names

    lora = bool(getattr(eng.model, "lora", False))
    if lora:
        w = {**w, **{n: t.to(torch.bfloat16) for n, t in eng.model.lora_init.items()}}
    sel = trainable_param_names(cfg, tcfg, getattr(eng.model, "n_tenants", 1))
    orc = TickOracle(cfg, w, tcfg, sel, device=device)
    orb = TickOracle(cfg, w, tcfg, sel, device=device, emulate_bf16=True)
    st = dict(ticks=0, tokens=0, ties=0, ft_ticks=0, pairs=0, first_steps=0, worst_logit_rel=0.0,
              worst_logit_rel_bf16emu=0.0, dL_rms=0.0, dL_rms_bf16emu=0.0, dm_rms=0.0, dm_rms_bf16emu=0.0,
              worst_dL_rel=0.0, worst_grad_rel=0.0, worst_grad_rel_bf16emu=0.0, dw_bad_frac=0.0,
              dw_bad_frac_bf16emu=0.0, adamw_bit_exact=0, kinds=set())
    fails: list[str] = []
    dL_g, dL_b, dm_g, dm_b = [], [], [], []
    grel_g, grel_b, dwf_g, dwf_b = [], [], [], []
    by_name: dict[str, list] = {}
    pre = (torch.cat([w[n].float().reshape(-1).cpu() for n in sel]).numpy(), None, None)
    pre = (pre[0], np.zeros_like(pre[0]), np.zeros_like(pre[0]))
    step = 0
    for rec in eng.records:
        b = rec["batch"]
        st["ticks"] += 1
        st["kinds"] |= set(b.seqs[:, 0].tolist())
        toks = rec["dec_tokens"] if rec["dec_tokens"] is not None else []
        # gradients at the DEVICE's margins (the DPO outer derivative is a function of the margin, whose bf16
        # forward noise is checked separately): the gradient comparison then measures the backward alone
        fm = rec.get("ft_margin")
        logits, ft = orc.run_tick(b, toks, rec["kept_post"], ft_margins=fm)
        logits_b, ft_b = orb.run_tick(b, toks, rec["kept_post"], ft_margins=fm)
        if b.n_dec:
            g = rec["dec_logits"]
            rel, relb = _rel(g, logits), _rel(logits_b, logits)
            st["worst_logit_rel"] = max(st["worst_logit_rel"], rel)
            st["worst_logit_rel_bf16emu"] = max(st["worst_logit_rel_bf16emu"], relb)
            if rel > max(1e-2, 1.5 * relb):
                fails.append(f"tick {rec['tick']}: logits rel-L2 {rel:.3e} (bf16 emulation {relb:.3e})")
            top2 = logits.topk(2, dim=-1).values
            gap = (top2[:, 0] - top2[:, 1]).numpy()
            for i, (a, t) in enumerate(zip(logits.argmax(-1).numpy(), toks)):
                st["tokens"] += 1
                if a != t:
                    st["ties"] += 1
                    if gap[i] >= 0.05:
                        fails.append(f"tick {rec['tick']} row {i}: token {t} != oracle {a} (gap {gap[i]:.3f})")
        if ft is None:
            continue
        st["ft_ticks"] += 1
        (losses, margins, grads), (losses_b, margins_b, grads_b) = ft, ft_b
        for i in range(len(losses)):
            st["pairs"] += 1
            g_lp, g_ref = rec["ft_lp"][i], rec["ref_lp"][i]
            L, Lg, Lb = losses[i], float(rec["ft_loss"][i]), losses_b[i]
            m, mg, mb = margins[i], float(rec["ft_margin"][i]), margins_b[i]
            if g_lp[0] == g_ref[0] and g_lp[1] == g_ref[1]:  # pi_theta == pi_ref for this pair
                st["first_steps"] += 1
                if mg != 0.0 or abs(Lg - math.log(2.0)) > 1e-7:
                    fails.append(f"tick {rec['tick']}: pi_theta == pi_ref but margin {mg}, loss {Lg}")
                continue
            dL_g.append(Lg - L)
            dL_b.append(Lb - L)
            dm_g.append(mg - m)
            dm_b.append(mb - m)
            st["worst_dL_rel"] = max(st["worst_dL_rel"], abs(Lg - L) / max(1.0, abs(L)))
        gflat = []
        for n in sel:
            gg, go, gb = rec["grad"][n].float(), grads[n].float(), grads_b[n].float()
            gflat.append(gg.reshape(-1))
            rel, relb = _rel(gg, go), _rel(gb, go)
            st["worst_grad_rel"] = max(st["worst_grad_rel"], rel)
            st["worst_grad_rel_bf16emu"] = max(st["worst_grad_rel_bf16emu"], relb)
            grel_g.append(rel)
            grel_b.append(relb)
            by_name.setdefault(n, []).append((rel, relb))
        # ---- AdamW in situ: bit-exact from the device's own pre-update state and gradient
        step += 1
        post = (rec["master"].numpy(), rec["adam_m"].numpy(), rec["adam_v"].numpy())
        if lora:
            widths = [(rec["grad"][n].shape[1], rec["grad"][n].numel()) for n in sel]
            want = adamw_np_tenants(pre, torch.cat(gflat).numpy(), rec["tenants"], rec["tenant_steps"], widths,
                                    tcfg.lora_rank, tcfg)
        else:
            want = adamw_np(*pre, torch.cat(gflat).numpy(), tcfg.lr, tcfg.beta1, tcfg.beta2, tcfg.eps,
                            tcfg.weight_decay, step)
        if all(np.array_equal(a.view(np.int32), b_.view(np.int32)) for a, b_ in zip(want, post)):
            st["adamw_bit_exact"] += 1
        else:
            fails.append(f"tick {rec['tick']}: AdamW not bit-exact with the fp32 restatement")
        # ---- updated weights vs the fp32 oracle's AdamW on its own gradient, same pre-update state
        bad = badb = tot = 0
        off = 0
        for n in sel:
            k = rec["grad"][n].numel()
            w0 = torch.from_numpy(pre[0][off: off + k])
            dw_o = orc.ex.master[n].reshape(-1).cpu() - w0
            tol = 1e-2 * dw_o.abs().max() + torch.from_numpy(np.abs(np.spacing(pre[0][off: off + k])))
            bad += int(((torch.from_numpy(post[0][off: off + k]) - w0 - dw_o).abs() > tol).sum())
            badb += int(((orb.ex.master[n].reshape(-1).cpu() - w0 - dw_o).abs() > tol).sum())
            tot += k
            off += k
        dwf_g.append(bad / tot)
        dwf_b.append(badb / tot)
        pre = post
        for o in (orc, orb):
            o.ex.load_state(rec["master"], rec["adam_m"], rec["adam_v"])
    rms = lambda v: float(np.sqrt(np.mean(np.square(v)))) if v else 0.0  # noqa: E731
    st["dL_rms"], st["dL_rms_bf16emu"], st["dm_rms"], st["dm_rms_bf16emu"] = rms(dL_g), rms(dL_b), rms(dm_g), rms(dm_b)
    st["grad_rel_rms"], st["grad_rel_rms_bf16emu"] = rms(grel_g), rms(grel_b)
    st["worst_grad_rel"], st["worst_grad_rel_bf16emu"] = max(grel_g, default=0.0), max(grel_b, default=0.0)
    st["dw_bad_frac"] = float(np.mean(dwf_g)) if dwf_g else 0.0
    st["dw_bad_frac_bf16emu"] = float(np.mean(dwf_b)) if dwf_b else 0.0
    if st["grad_rel_rms"] > 1.5 * st["grad_rel_rms_bf16emu"] + 2e-3:
        fails.append(f"selected-grad rel-L2 rms {st['grad_rel_rms']:.3e} vs bf16 emulation {st['grad_rel_rms_bf16emu']:.3e}")
    if st["worst_grad_rel"] > max(2.0 * st["worst_grad_rel_bf16emu"], 0.02):
        fails.append(f"worst selected-grad rel-L2 {st['worst_grad_rel']:.3e} vs bf16 emulation "
                     f"{st['worst_grad_rel_bf16emu']:.3e}")
    if st["dw_bad_frac"] > 1.5 * st["dw_bad_frac_bf16emu"] + 1e-3:
        fails.append(f"mean fraction of updated weights outside the bound {st['dw_bad_frac']:.3e} vs bf16 emulation "
                     f"{st['dw_bad_frac_bf16emu']:.3e}")
    # the per-pair loss / margin errors of both implementations are draws of bf16 noise: the ratio of their rms over
    # n pairs is sqrt(F(n, n))-distributed, so few-pair samples get the 99.5% quantile instead of the flat 1.5
    # (below 20 pairs the rms of either sample is too uncertain to rank two noise sources -- sqrt(F_0.995) > 1.8 --
    # so only the per-pair absolute backstop below applies)
    n_pairs = len(dm_g)
    ratio = max(1.5, float(np.sqrt(f_dist.ppf(0.995, n_pairs, n_pairs)))) if n_pairs >= 20 else None
    st["pair_rms_ratio_bound"] = ratio
    if ratio is not None and st["dL_rms"] > ratio * st["dL_rms_bf16emu"] + 1e-3:
        fails.append(f"DPO loss rms error {st['dL_rms']:.3e} vs bf16 emulation {st['dL_rms_bf16emu']:.3e} (x{ratio:.2f})")
    if ratio is not None and st["dm_rms"] > ratio * st["dm_rms_bf16emu"] + 1e-3:
        fails.append(f"DPO margin rms error {st['dm_rms']:.3e} vs bf16 emulation {st['dm_rms_bf16emu']:.3e} (x{ratio:.2f})")
    # absolute backstop for every pair: the margin within 0.5 nat of the fp32 oracle, the loss (1-Lipschitz in the
    # margin at beta <= 1) within that pair's margin error
    st["worst_dm"] = max((abs(x) for x in dm_g), default=0.0)
    st["worst_dm_bf16emu"] = max((abs(x) for x in dm_b), default=0.0)
    if st["worst_dm"] > max(0.5, 2.0 * st["worst_dm_bf16emu"]):
        fails.append(f"a DPO margin is {st['worst_dm']:.3f} nat from the fp32 oracle (bf16 emulation's worst "
                     f"{st['worst_dm_bf16emu']:.3f})")
    if any(abs(a) > max(1.0, tcfg.dpo_beta) * abs(b_) + 1e-3 for a, b_ in zip(dL_g, dm_g)):
        fails.append("a DPO loss error exceeds its margin error (the loss is beta-Lipschitz in the margin)")
    if st["tokens"] and st["ties"] > max_tie_frac * st["tokens"]:
        fails.append(f"{st['ties']} near-tie token exemptions of {st['tokens']}")
    st["kinds"] = sorted(st["kinds"])
    if fails:  # per-tensor worst (gpu, bf16 emulation) rel-L2, to localise a gradient failure
        st["grad_rel_worst_by_name"] = {n: (round(max(a for a, _ in v), 4), round(max(b_ for _, b_ in v), 4))
                                        for n, v in by_name.items()}
    print(f"parity {label}: " + ", ".join(f"{k}={v:.3g}" if isinstance(v, float) else f"{k}={v}" for k, v in st.items()))
    assert not fails, f"{label}: {len(fails)} parity failures, first: " + "; ".join(fails[:8]) + f" | stats {st}"
    return st
