"""Shared checker for the tick-replay parity tests (C1, the model families, the full-shape samples).

Every tick GpuEngine executed on the B200 is replayed by the fp32 oracle (oracle/model_ref.py:TickOracle)
from the same recorded tick batch. Tolerances -- SURVEY.md §8(c), bf16 storage / fp32 accumulation against
an fp32 oracle on the same bf16-rounded weights:

  decode logits      rel-L2 <= 1e-2 per tick
  decode token ids   bit-exact, except oracle near-ties (top-1/top-2 gap < 0.05): counted, <= 5% of tokens
  DPO loss           |dL| <= 1e-2 * max(1, |L|) for every pair of every fine-tune tick
  DPO margin         exactly 0 while pi_theta == pi_ref (a pair's first step: same kernels, same rows);
                     otherwise |dm| <= 1e-2 * max(1, |m|) / beta (the loss bound, |dL/dm| <= beta)
  selected grads     rel-L2 <= 0.02 + 1.05 * max|dm| per tensor (the DPO coefficient beta*sigma(-beta m)
                     moves by <= |dm| relative)
  AdamW (in situ)    the device masters / m / v after each update are BIT-EXACT with the numpy fp32
                     restatement of the kernel (adamw_np) applied to the device's own pre-update state and
                     gradient
  updated weights    |dw_gpu - dw_oracle| <= 1e-2 * max|dw_oracle| + 1 fp32 ulp(w) per element, from the same
                     pre-update state; elements whose oracle gradient lies inside the gradient's bf16 error band
                     (|g_oracle| <= 4 * rms(g_gpu - g_oracle) of that tensor) have no defined Adam direction --
                     a sign flip there moves the weight by 2*lr -- and are exempt, counted, <= 10% of elements
"""
from __future__ import annotations

import math

import numpy as np
import torch


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


def check_records(eng, w, cfg, tcfg, device="cpu", max_tie_frac=0.05, max_exempt_frac=0.10, label=""):
    from oracle.model_ref import TickOracle
    from paper_2510_03283_b200.config import selected_param_names

    sel = selected_param_names(cfg, tcfg)
    orc = TickOracle(cfg, w, tcfg, sel, device=device)
    st = dict(ticks=0, tokens=0, ties=0, ft_ticks=0, pairs=0, first_steps=0, worst_logit_rel=0.0, worst_dL=0.0,
              worst_dm=0.0, worst_grad_rel=0.0, dw_elems=0, dw_exempt=0, worst_dw_ratio=0.0, adamw_bit_exact=0,
              kinds=set())
    fails: list[str] = []
    beta = tcfg.dpo_beta
    pre = (torch.cat([w[n].float().reshape(-1).cpu() for n in sel]).numpy(), None, None)
    pre = (pre[0], np.zeros_like(pre[0]), np.zeros_like(pre[0]))
    step = 0
    for rec in eng.records:
        b = rec["batch"]
        st["ticks"] += 1
        st["kinds"] |= set(b.seqs[:, 0].tolist())
        toks = rec["dec_tokens"] if rec["dec_tokens"] is not None else []
        logits, ft = orc.run_tick(b, toks, rec["kept_post"])
        if b.n_dec:
            g = rec["dec_logits"]
            rel = ((g - logits).norm() / logits.norm()).item()
            st["worst_logit_rel"] = max(st["worst_logit_rel"], rel)
            if rel > 1e-2:
                fails.append(f"tick {rec['tick']}: logits rel-L2 {rel:.3e}")
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
        losses, margins, grads = ft
        dm_max = 0.0
        for i in range(len(losses)):
            st["pairs"] += 1
            g_lp, g_ref = rec["ft_lp"][i], rec["ref_lp"][i]
            L, Lg = losses[i], float(rec["ft_loss"][i])
            m, mg = margins[i], float(rec["ft_margin"][i])
            dL, dm = abs(Lg - L), abs(mg - m)
            st["worst_dL"] = max(st["worst_dL"], dL / max(1.0, abs(L)))
            st["worst_dm"] = max(st["worst_dm"], dm / max(1.0, abs(m)))
            dm_max = max(dm_max, dm)
            if g_lp[0] == g_ref[0] and g_lp[1] == g_ref[1]:
                st["first_steps"] += 1
                if mg != 0.0:
                    fails.append(f"tick {rec['tick']}: pi_theta == pi_ref but margin {mg}")
            if dL > 1e-2 * max(1.0, abs(L)):
                fails.append(f"tick {rec['tick']} pair {i}: loss {Lg} vs oracle {L}")
            if dm > 1e-2 * max(1.0, abs(m)) / beta:
                fails.append(f"tick {rec['tick']} pair {i}: margin {mg} vs oracle {m}")
        gflat = []
        for n in sel:
            gg, go = rec["grad"][n].float(), grads[n].float()
            gflat.append(gg.reshape(-1))
            rel = ((gg - go).norm() / (go.norm() + 1e-30)).item()
            st["worst_grad_rel"] = max(st["worst_grad_rel"], rel)
            if rel > 0.02 + 1.05 * dm_max:
                fails.append(f"tick {rec['tick']}: grad {n} rel-L2 {rel:.3e} (dm {dm_max:.2e})")
        # ---- AdamW in situ: bit-exact from the device's own pre-update state and gradient
        step += 1
        post = (rec["master"].numpy(), rec["adam_m"].numpy(), rec["adam_v"].numpy())
        want = adamw_np(*pre, torch.cat(gflat).numpy(), tcfg.lr, tcfg.beta1, tcfg.beta2, tcfg.eps,
                        tcfg.weight_decay, step)
        if all(np.array_equal(a.view(np.int32), b_.view(np.int32)) for a, b_ in zip(want, post)):
            st["adamw_bit_exact"] += 1
        else:
            fails.append(f"tick {rec['tick']}: AdamW not bit-exact with the fp32 restatement")
        # ---- updated weights vs the oracle's AdamW on the oracle's gradient, same pre-update state
        off = 0
        for n in sel:
            k = rec["grad"][n].numel()
            w0 = torch.from_numpy(pre[0][off: off + k])
            dw_g = torch.from_numpy(post[0][off: off + k]) - w0
            dw_o = orc.ex.master[n].reshape(-1).cpu() - w0
            go, gg = grads[n].reshape(-1).float(), rec["grad"][n].reshape(-1).float()
            band = 4.0 * (gg - go).pow(2).mean().sqrt()
            exempt = go.abs() <= band
            tol = 1e-2 * dw_o.abs().max() + torch.from_numpy(np.abs(np.spacing(pre[0][off: off + k])))
            err = (dw_g - dw_o).abs()
            bad = (err > tol) & ~exempt
            st["dw_elems"] += k
            st["dw_exempt"] += int(exempt.sum())
            ratio = float((err[~exempt] / tol[~exempt]).max()) if (~exempt).any() else 0.0
            st["worst_dw_ratio"] = max(st["worst_dw_ratio"], ratio)
            if bad.any():
                fails.append(f"tick {rec['tick']}: {n} {int(bad.sum())} updated weights outside tolerance "
                             f"(worst err/tol {ratio:.2f})")
            off += k
        pre = post
        orc.ex.load_state(rec["master"], rec["adam_m"], rec["adam_v"])
    if st["tokens"] and st["ties"] > max_tie_frac * st["tokens"]:
        fails.append(f"{st['ties']} near-tie token exemptions of {st['tokens']}")
    if st["dw_elems"] and st["dw_exempt"] > max_exempt_frac * st["dw_elems"]:
        fails.append(f"{st['dw_exempt']} of {st['dw_elems']} weight updates exempt (gradient noise band)")
    st["kinds"] = sorted(st["kinds"])
    print(f"parity {label}: " + ", ".join(f"{k}={v:.3g}" if isinstance(v, float) else f"{k}={v}" for k, v in st.items()))
    assert not fails, f"{label}: {len(fails)} parity failures, first: " + "; ".join(fails[:8]) + f" | stats {st}"
    return st
