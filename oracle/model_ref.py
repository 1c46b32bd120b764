"""CPU ORACLE (test infrastructure only) for the model arithmetic of MACE's hybrid iteration.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module. It is
the checker, never the thing measured or shipped; the product path (paper_2510_03283_b200) never
imports it.

PARITY STATUS: the reference (macesim) is a simulator with no logits, tokens, gradients or weights
(SURVEY.md §0.3, §8(c)), so the model arithmetic here is *parity unpinned* against the reference
itself. It is a plain fp32 PyTorch restatement of standard definitions, pinned where the reference
has arithmetic:
  * DPO scalar stage  = macesim.alignment.dpo_loss (alignment.py:39-47), pinned by golden vectors
    generated from the reference (tests/golden/dpo_golden.json, tests/golden/make_golden.py).
  * tick / row order  = Engine._execute (engine.py:573-676): prefills in trie-DFS order, decodes
    and fine-tunes by id (engine.py:578-584).
  * KV semantics      = cache.py:67-273 + engine.py:496-529: prompt KV is never pruned; decode slots
    are trimmed oldest-first per KV head to the reference's kept[h] counts.
  * pi_ref frozen at init; AdamW = torch.optim.AdamW's update order.
Builder-defined (no reference exists, documented in DESIGN.md): the decoder shapes, synthetic
chosen/rejected token content, the selected-parameter rule (top-k layers + final norm), AdamW
hyper-parameters, and the decode token convention (prefill writes the prompt KV and emits no token,
engine.py:474 / test_engine.py:33-36; decode step k consumes x_k at position P-2+k with
x_1 = prompt[-1], x_k = y_{k-1}).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F


# ----------------------------------------------------------------------------- scalar DPO stage
def dpo_loss_scalar(margin: float, beta: float) -> float:
    """-log sigmoid(beta*m), the reference's stable form (alignment.py:39-47)."""
    if beta <= 0:
        raise ValueError("beta must be > 0")
    x = -beta * margin
    if x > 0:
        return x + math.log1p(math.exp(-x))
    return math.log1p(math.exp(x))


# ----------------------------------------------------------------------------- building blocks
def rms_norm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def layer_norm(x, w, b, eps):
    mu = x.mean(-1, keepdim=True)
    var = (x - mu).pow(2).mean(-1, keepdim=True)
    return (x - mu) * torch.rsqrt(var + eps) * w + b


def gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


def rope(x, pos, theta):
    """x [n, H, hd]; rotate-half convention (Llama); pos int64 [n]."""
    hd = x.shape[-1]
    inv = theta ** (-torch.arange(0, hd // 2, dtype=torch.float64, device=x.device) * 2.0 / hd)
    ang = pos.to(x.device, torch.float64)[:, None] * inv[None, :]
    cos = torch.cos(ang).to(x.dtype)[:, None, :]
    sin = torch.sin(ang).to(x.dtype)[:, None, :]
    x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


@dataclass
class _Seq:
    prompt: list[int]
    k_prompt: list = field(default_factory=list)   # per layer [P, Hkv, hd]
    v_prompt: list = field(default_factory=list)
    k_dec: list = field(default_factory=list)      # per layer list of [Hkv, hd]
    v_dec: list = field(default_factory=list)


class OracleModel:
    """fp32 CPU decoder: Llama (RMSNorm/RoPE/GQA/SwiGLU) or GPT-2 (LayerNorm/learned pos/GELU/bias)."""

    def __init__(self, cfg, weights: dict[str, torch.Tensor], device: str | torch.device = "cpu", lora_rank: int = 0,
                 lora_scale: float = 0.0):
        self.cfg = cfg
        self.dev = torch.device(device)
        self.w = {k: v.detach().to(self.dev, torch.float32).clone() for k, v in weights.items()}
        # per-tenant LoRA (weights hold "lora.{l}.a_{p}" [R, in] / "lora.{l}.bt_{p}" [R, out], tenants stacked)
        self.lora_rank, self.lora_scale = lora_rank, lora_scale

    def _adapter(self, X, l, proj, params, tenant):
        """(alpha / r) * mask_tenant(X A^T) B^T: each row uses only its own tenant's rank-r block (LoRA,
        PAPER.md:440-441); tenant None (pi_ref, the frozen base model) -> no adapter."""
        key = f"lora.{l}.a_{proj}"
        if tenant is None or not self.lora_rank or key not in params:
            return None
        A, Bt = params[key], params[f"lora.{l}.bt_{proj}"]
        Z = X @ A.t()
        cols = torch.arange(A.shape[0], device=X.device) // self.lora_rank
        mask = (cols[None, :] == tenant[:, None]).to(Z.dtype)
        return self._round_z(self.lora_scale * Z * mask) @ Bt

    def _round_z(self, z):
        return z

    # -- one decoder layer over rows x [n, d]; kv_ctx(l, k_new, v_new) -> (K [m,Hkv,hd], V, mask [n,Hkv?,m])
    def _norm(self, x, name, params):
        c = self.cfg
        if c.family == "llama":
            return rms_norm(x, params[name + ".w"], c.norm_eps)
        return layer_norm(x, params[name + ".w"], params[name + ".b"], c.norm_eps)

    def _lin(self, x, name, params, extra=None):
        y = x @ params[name + ".w"].t()
        if extra is not None:
            y = y + extra
        if self.cfg.has_bias:
            y = y + params[name + ".b"]
        return y

    def embed(self, tokens, pos, params=None):
        params = params or self.w
        x = params["embed"][torch.as_tensor(tokens, dtype=torch.long, device=self.dev)]
        if self.cfg.family == "gpt2":
            x = x + params["pos_embed"][torch.as_tensor(pos, dtype=torch.long, device=self.dev)]
        return x

    def layer(self, l, x, pos, attend, params=None, tenant=None):
        """attend(l, q[n,Hq,hd], k[n,Hkv,hd], v) -> o [n, Hq, hd]; tenant: LongTensor [n] (LoRA rows) or None"""
        c = self.cfg
        params = params or self.w
        p = f"layers.{l}."
        h = self._norm(x, p + "attn_norm", params)
        qkv = self._lin(h, p + "qkv", params, self._adapter(h, l, "qkv", params, tenant))
        Hq, Hk, hd = c.n_heads, c.n_kv_heads, c.head_dim
        q = qkv[:, : Hq * hd].reshape(-1, Hq, hd)
        k = qkv[:, Hq * hd: (Hq + Hk) * hd].reshape(-1, Hk, hd)
        v = qkv[:, (Hq + Hk) * hd:].reshape(-1, Hk, hd)
        if c.family == "llama":
            pos_t = torch.as_tensor(pos, dtype=torch.long, device=self.dev)
            q = rope(q, pos_t, c.rope_theta)
            k = rope(k, pos_t, c.rope_theta)
        o = attend(l, q, k, v).reshape(-1, Hq * hd)
        x = x + self._lin(o, p + "o", params)
        ad = self._adapter(o, l, "o", params, tenant)
        if ad is not None:
            x = x + ad
        h = self._norm(x, p + "mlp_norm", params)
        u = self._lin(h, p + "up", params, self._adapter(h, l, "up", params, tenant))
        if c.family == "llama":
            a = F.silu(u[:, : c.ffn]) * u[:, c.ffn:]
        else:
            a = gelu_tanh(u)
        x = x + self._lin(a, p + "down", params)
        ad = self._adapter(a, l, "down", params, tenant)
        return x if ad is None else x + ad

    def final(self, x, params=None):
        params = params or self.w
        return self._norm(x, "final_norm", params) @ params["embed"].t()

    def attention(self, q, K, V, mask):
        """q [n,Hq,hd], K/V [m,Hkv,hd] or per-head lists, mask bool [n, Hkv, m] (True = attend)."""
        c = self.cfg
        g = c.group
        Kx = K.repeat_interleave(g, dim=1)  # [m, Hq, hd]
        Vx = V.repeat_interleave(g, dim=1)
        s = torch.einsum("nhd,mhd->nhm", q, Kx) / math.sqrt(c.head_dim)
        mk = mask.repeat_interleave(g, dim=1)
        s = s.masked_fill(~mk, float("-inf"))
        p = torch.softmax(s, dim=-1)
        return torch.einsum("nhm,mhd->nhd", p, Vx)

    # -- full causal sequence (prefill, fine-tune); returns hidden [n, d] and per-layer (k, v)
    def forward_seq(self, tokens, pos0=0, params=None, collect_kv=False, tenant=None):
        n = len(tokens)
        if tenant is not None:
            tenant = torch.full((n,), int(tenant), dtype=torch.long, device=self.dev)
        pos = list(range(pos0, pos0 + n))
        x = self.embed(tokens, pos, params)
        causal = torch.tril(torch.ones(n, n, dtype=torch.bool, device=self.dev))
        kvs = []

        def attend(l, q, k, v):
            if collect_kv:
                kvs.append((k.detach().clone(), v.detach().clone()))
            mask = causal[:, None, :].expand(n, self.cfg.n_kv_heads, n)
            return self.attention(q, k, v, mask)

        for l in range(self.cfg.n_layers):
            x = self.layer(l, x, pos, attend, params, tenant)
        return x, kvs

    def seq_logprob(self, prompt, response, params=None, tenant=None):
        """Sum of log p(response | prompt) under ``params`` (and the tenant's adapter, LoRA); response token i
        predicted at P+i-1."""
        toks = list(prompt) + list(response)
        h, _ = self.forward_seq(toks, params=params, tenant=tenant)
        P = len(prompt)
        logits = self.final(h[P - 1: P - 1 + len(response)], params)
        lp = torch.log_softmax(logits, dim=-1)
        tgt = torch.as_tensor(response, dtype=torch.long, device=self.dev)
        return lp.gather(1, tgt[:, None]).sum()


class Bf16EmulationModel(OracleModel):
    """The same restatement with every GEMM / attention operand and output rounded to bf16 where the B200 path
    stores bf16 (norm outputs, projections, attention q/k/v and output, lm_head input) and the residual stream,
    norm statistics and softmax kept in fp32 -- an INDEPENDENT bf16 implementation (torch) of the same numerics
    class. The parity tests use its distance to the fp32 oracle as the noise floor of bf16 arithmetic: the
    device must be no further from fp32 than this (tests/parity_util.py). Autograd through the casts rounds the
    backward's activations gradients to bf16 as well."""

    def _lin(self, x, name, params, extra=None):
        y = (x.to(torch.bfloat16) @ params[name + ".w"].to(torch.bfloat16).t()).float()
        if extra is not None:
            y = y + extra
        if self.cfg.has_bias:
            y = y + params[name + ".b"]
        return y.to(torch.bfloat16).float()

    def _norm(self, x, name, params):
        return super()._norm(x, name, params).to(torch.bfloat16).float()

    def _round_z(self, z):
        return z.to(torch.bfloat16).float()

    def attention(self, q, K, V, mask):
        r = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
        return r(super().attention(r(q), r(K), r(V), mask))

    def final(self, x, params=None):
        params = params or self.w
        return self._norm(x, "final_norm", params) @ params["embed"].to(torch.bfloat16).float().t()


class OracleExecutor:
    """Request-level restatement of the GPU hybrid step (prefill / decode / DPO fine-tune)."""

    def __init__(self, cfg, weights, tcfg, selected_names, device: str | torch.device = "cpu", emulate_bf16=False):
        self.cfg = cfg
        self.tcfg = tcfg
        self.lora_rank = getattr(tcfg, "lora_rank", None) or 0
        self.model = (Bf16EmulationModel if emulate_bf16 else OracleModel)(
            cfg, weights, device, self.lora_rank, tcfg.lora_alpha / self.lora_rank if self.lora_rank else 0.0)
        self.selected = list(selected_names)
        # pi_ref frozen at init; LoRA: pi_ref is the frozen base model (every adapter off)
        self.ref_params = {} if self.lora_rank else {n: self.model.w[n].clone() for n in self.selected}
        self.tenant_steps: dict[int, int] = {}
        self.master = {n: self.model.w[n].clone() for n in self.selected}
        self.m = {n: torch.zeros_like(self.master[n]) for n in self.selected}
        self.v = {n: torch.zeros_like(self.master[n]) for n in self.selected}
        self.step = 0
        self.seqs: dict[int, _Seq] = {}
        self.ref_lp_cache: dict[int, tuple[float, float]] = {}

    # ---------------------------------------------------------------- inference rows
    def prefill(self, rid: int, prompt: list[int]) -> None:
        """Engine._exec_prefill (engine.py:444-480): prompt KV for all P tokens, no token emitted."""
        _, kvs = self.model.forward_seq(prompt, collect_kv=True)
        s = _Seq(prompt=list(prompt))
        s.k_prompt = [k for k, _ in kvs]
        s.v_prompt = [v for _, v in kvs]
        s.k_dec = [[] for _ in range(self.cfg.n_layers)]
        s.v_dec = [[] for _ in range(self.cfg.n_layers)]
        self.seqs[rid] = s

    def decode(self, rid: int, x_token: int, kept_pre: list[int] | None) -> torch.Tensor:
        """Engine._exec_decode (engine.py:482-532) step k: returns logits [V] for y_k.

        Window for KV head h = prompt[:P-1] (never pruned) + the last kept_pre[h] decode slots + the
        new slot k. ``kept_pre`` None means no pruning (all decode slots).
        """
        s = self.seqs[rid]
        c = self.cfg
        P = len(s.prompt)
        k_idx = len(s.k_dec[0]) + 1          # this is decode slot k (1-based)
        pos = P - 2 + k_idx
        x = self.model.embed([x_token], [pos])

        def attend(l, q, k, v):
            s.k_dec[l].append(k[0].clone())
            s.v_dec[l].append(v[0].clone())
            Kp = s.k_prompt[l][: P - 1]
            Vp = s.v_prompt[l][: P - 1]
            Kd = torch.stack(s.k_dec[l])   # [k, Hkv, hd]
            Vd = torch.stack(s.v_dec[l])
            K = torch.cat([Kp, Kd])
            V = torch.cat([Vp, Vd])
            m = K.shape[0]
            mask = torch.zeros(1, c.n_kv_heads, m, dtype=torch.bool, device=K.device)
            mask[:, :, : P - 1] = True
            for h in range(c.n_kv_heads):
                keep = (k_idx - 1) if kept_pre is None else min(kept_pre[h], k_idx - 1)
                lo = (P - 1) + (k_idx - 1 - keep)
                mask[0, h, lo:] = True
            return self.model.attention(q, K, V, mask)

        for l in range(c.n_layers):
            x = self.model.layer(l, x, [pos], attend)
        return self.model.final(x)[0]

    def release(self, rid: int) -> None:
        self.seqs.pop(rid, None)

    # ---------------------------------------------------------------- fine-tune rows
    def dpo_step(self, pairs: list[tuple[int, list[int], list[int], list[int]]], coef_margins=None):
        """One optimizer step on mean_i softplus(-beta * m_i) over the tick's FT pairs.

        pairs: (rid, prompt, chosen, rejected[, tenant]). m_i = (lp_c - ref_c) - (lp_r - ref_r) with ref log-probs
        under the frozen pi_ref, computed once per pair (alignment.py:39-47 for the scalar stage). LoRA: the policy
        runs with the pair's tenant adapter, pi_ref without adapters.
        coef_margins: when given (the device's per-pair margins), the gradient is taken at THOSE margins -- the
        loss's outer derivative -beta * sigma(-beta * m_i) / n uses m_i = coef_margins[i] -- so a gradient comparison
        isolates the backward from the forward's margin rounding noise (the reported losses / margins stay the
        oracle's own).
        Returns per-pair (loss, margin) and the gradients of the selected parameters.
        """
        beta = self.tcfg.dpo_beta
        params = dict(self.model.w)
        for n in self.selected:
            params[n] = self.model.w[n].clone().requires_grad_(True)
        ref = dict(self.model.w)
        ref.update(self.ref_params)
        losses, margins, total = [], [], 0.0
        self.last_lp = []
        for pr in pairs:
            rid, prompt, chosen, rejected = pr[:4]
            ten = (pr[4] if len(pr) > 4 else 0) if self.lora_rank else None
            if rid not in self.ref_lp_cache:
                with torch.no_grad():
                    self.ref_lp_cache[rid] = (
                        float(self.model.seq_logprob(prompt, chosen, ref)),
                        float(self.model.seq_logprob(prompt, rejected, ref)),
                    )
            rc, rr = self.ref_lp_cache[rid]
            lc = self.model.seq_logprob(prompt, chosen, params, tenant=ten)
            lr_ = self.model.seq_logprob(prompt, rejected, params, tenant=ten)
            m = (lc - rc) - (lr_ - rr)
            loss = F.softplus(-beta * m)
            if coef_margins is None:
                total = total + loss / len(pairs)
            else:  # d softplus(-beta m) / dm at the given margin, times m (a surrogate with that gradient)
                mi = float(coef_margins[len(losses)])
                total = total + (-beta * torch.sigmoid(torch.tensor(-beta * mi, dtype=m.dtype))) * m / len(pairs)
            losses.append(float(loss.detach()))
            margins.append(float(m.detach()))
            self.last_lp.append((float(lc.detach()), float(lr_.detach()), rc, rr))
        total.backward()
        grads = {n: params[n].grad.detach().clone() for n in self.selected}
        return losses, margins, grads

    def load_state(self, master_flat, m_flat, v_flat) -> None:
        """Adopt the device's optimizer state (flat fp32, selected-name order) so the next tick compares
        one step from identical weights instead of two drifting trajectories."""
        off = 0
        for n in self.selected:
            k = self.master[n].numel()
            shape = self.master[n].shape
            dev = self.model.dev
            self.master[n] = master_flat[off: off + k].view(shape).to(dev).clone()
            self.m[n] = m_flat[off: off + k].view(shape).to(dev).clone()
            self.v[n] = v_flat[off: off + k].view(shape).to(dev).clone()
            self.model.w[n] = self.master[n].to(torch.bfloat16).float()
            off += k

    def adamw(self, grads: dict[str, torch.Tensor], tenants=None) -> None:
        """torch.optim.AdamW update order on fp32 masters; working weights = bf16(master). LoRA: one optimizer per
        tenant -- only the stepping tenants' adapter rows move, each with its own step count."""
        t = self.tcfg
        if self.lora_rank:
            r = self.lora_rank
            for u in sorted(set(tenants or [])):
                k = self.tenant_steps[u] = self.tenant_steps.get(u, 0) + 1
                bc1, bc2 = 1.0 - t.beta1 ** k, 1.0 - t.beta2 ** k
                rows = slice(u * r, (u + 1) * r)
                for n in self.selected:
                    adamw_reference(self.master[n][rows], self.m[n][rows], self.v[n][rows], grads[n][rows], t.lr,
                                    t.beta1, t.beta2, t.eps, t.weight_decay, bc1, bc2)
                    self.model.w[n] = self.master[n].to(torch.bfloat16).float()
            return
        self.step += 1
        bc1 = 1.0 - t.beta1 ** self.step
        bc2 = 1.0 - t.beta2 ** self.step
        for n in self.selected:
            adamw_reference(self.master[n], self.m[n], self.v[n], grads[n], t.lr, t.beta1, t.beta2, t.eps,
                            t.weight_decay, bc1, bc2)
            self.model.w[n] = self.master[n].to(torch.bfloat16).float()


def adamw_reference(p, m, v, g, lr, b1, b2, eps, wd, bc1, bc2):
    """In-place fp32 AdamW restatement (torch.optim.AdamW single-tensor order)."""
    p.mul_(1.0 - lr * wd)
    m.lerp_(g, 1.0 - b1)
    v.mul_(b2).addcmul_(g, g, value=1.0 - b2)
    step_size = lr / bc1
    denom = (v.sqrt() / math.sqrt(bc2)).add_(eps)
    p.addcdiv_(m, denom, value=-step_size)


class TickOracle:
    """Replays the GPU's recorded tick batches (same rows, same page tables, same windows) in fp32.

    The tick batch is the *input format* (row order, prompt page tables, copy-on-diverge list,
    decode windows): the oracle reads it the way the device does, so prefix KV shared through the
    trie is the KV the sharing request actually sees (computed by whichever earlier prefill, under
    the weights of that time), exactly like the device pages.

    ``device``: where the fp32 restatement executes. CPU for the small configs; the full-shape sampled
    replays of Llama-3.2-1B / Llama-3-8B (tests/test_parity_shapes_gpu.py) run the SAME fp32 code through
    torch on the GPU (cuBLAS fp32 with TF32 disabled -- an independent implementation from the product's
    bf16 tcgen05 kernels), because a CPU fp32 replay of an 8B model exceeds the test budget.
    """

    PAGE = 16

    def __init__(self, cfg, weights, tcfg, selected_names, device: str | torch.device = "cpu", emulate_bf16=False):
        self.cfg = cfg
        self.dev = torch.device(device)
        self.ex = OracleExecutor(cfg, weights, tcfg, selected_names, self.dev, emulate_bf16)
        self.model = self.ex.model
        L, H, hd = cfg.n_layers, cfg.n_kv_heads, cfg.head_dim
        self._shape = (L, H, self.PAGE, hd)
        # prompt page groups: group id -> row of a dense store [n, L, H, 16, hd] (grown on demand)
        self.gslot: dict[int, int] = {}
        self.kstore = torch.zeros((0,) + self._shape, device=self.dev)
        self.vstore = torch.zeros((0,) + self._shape, device=self.dev)
        self.ptab: dict[int, list[int]] = {}
        self.dec: dict[int, dict] = {}
        self.last_token: dict[int, int] = {}

    def _slots(self, groups: list[int]) -> torch.Tensor:
        """Store rows of the given groups (new groups get zero pages, like the device's zeroed pool)."""
        new = [g for g in dict.fromkeys(groups) if g not in self.gslot]
        if new:
            n0 = self.kstore.shape[0]
            for i, g in enumerate(new):
                self.gslot[g] = n0 + i
            z = torch.zeros((len(new),) + self._shape, device=self.dev)
            self.kstore = torch.cat([self.kstore, z])
            self.vstore = torch.cat([self.vstore, z.clone()])
        return torch.tensor([self.gslot[g] for g in groups], dtype=torch.long, device=self.dev)

    def run_tick(self, batch, gpu_tokens, kept_post, ft_margins=None):
        """Returns (decode logits [n_dec, V], FT (losses, margins, grads) or None). ft_margins: the device's
        per-pair margins -- gradients are then taken at them (OracleExecutor.dpo_step coef_margins)."""
        c = self.cfg
        H, P16 = c.n_kv_heads, self.PAGE
        for slot, row in zip(batch.ptab_slots.tolist(), batch.ptab_rows.tolist()):
            self.ptab[slot] = row
        for src, dst, n, _ in batch.page_copies.tolist():
            si, di = self._slots([src, dst]).tolist()
            self.kstore[di, :, :, :n] = self.kstore[si, :, :, :n]
            self.vstore[di, :, :, :n] = self.vstore[si, :, :, :n]
        ft0 = batch.ft0
        seqs = batch.seqs.tolist()
        inf = [s for s in seqs if s[0] != 2]
        logits = None
        if ft0 > 0:
            toks = []
            for r in range(ft0):
                t = int(batch.tokens[r])
                toks.append(self.last_token[-t - 1] if t < 0 else t)
            pos = batch.pos[:ft0].tolist()
            x = self.model.embed(toks, pos)
            for s in inf:  # decode slot state (reset when a slot starts a new request)
                if s[0] == 1:
                    j = int(batch.row_kvi[s[1]])
                    if j == 0 or s[3] not in self.dec:
                        self.dec[s[3]] = {"k": [[] for _ in range(c.n_layers)], "v": [[] for _ in range(c.n_layers)],
                                          "first": [0] * H}
            # per prefill sequence: the (store row, page row) of each written prompt index and of each visible one
            wr, rd = {}, {}
            for s in inf:
                kind, q0, ql, slot, n_pv = s[:5]
                tab = self.ptab[slot]
                if kind == 0:
                    t = batch.row_kvi[q0: q0 + ql].astype(np.int64)
                    wr[q0] = (self._slots([tab[i] for i in (t // P16).tolist()]), torch.as_tensor(t % P16, device=self.dev))
                if n_pv:
                    t = np.arange(n_pv)
                    rd[q0] = (self._slots([tab[i] for i in (t // P16).tolist()]), torch.as_tensor(t % P16, device=self.dev))

            def attend(l, q, k, v):
                # 1) write this layer's K/V for every row (prefill -> pages, decode -> slot lists)
                for s in inf:
                    kind, q0, ql, slot, n_pv = s[:5]
                    if kind == 0:
                        gs, rr = wr[q0]
                        self.kstore[gs, l, :, rr] = k[q0: q0 + ql]
                        self.vstore[gs, l, :, rr] = v[q0: q0 + ql]
                    else:
                        d = self.dec[slot]
                        assert len(d["k"][l]) == int(batch.row_kvi[q0]), "decode slot index mismatch"
                        d["k"][l].append(k[q0].clone())
                        d["v"][l].append(v[q0].clone())
                # 2) attention per sequence over its visible KV
                o = torch.zeros(q.shape[0], c.n_heads, c.head_dim, device=self.dev)
                for s in inf:
                    kind, q0, ql, slot, n_pv = s[:5]
                    if n_pv:
                        gs, rr = rd[q0]
                        Kp, Vp = self.kstore[gs, l, :, rr], self.vstore[gs, l, :, rr]  # [n_pv, H, hd]
                    else:
                        Kp = Vp = torch.zeros(0, H, c.head_dim, device=self.dev)
                    if kind == 0:
                        m = n_pv
                        qlog = torch.arange(ql, device=self.dev)[:, None] + (n_pv - ql)
                        mask = (torch.arange(m, device=self.dev)[None, :] <= qlog)[:, None, :].expand(ql, H, m)
                        o[q0: q0 + ql] = self.model.attention(q[q0: q0 + ql], Kp, Vp, mask)
                    else:
                        d = self.dec[slot]
                        j = int(batch.row_kvi[q0])
                        K = torch.cat([Kp, torch.stack(d["k"][l])])
                        V = torch.cat([Vp, torch.stack(d["v"][l])])
                        mask = torch.zeros(1, H, K.shape[0], dtype=torch.bool, device=self.dev)
                        mask[:, :, :n_pv] = True
                        for h in range(H):
                            mask[0, h, n_pv + d["first"][h]: n_pv + j + 1] = True
                        o[q0: q0 + 1] = self.model.attention(q[q0: q0 + 1], K, V, mask)
                return o

            rt = getattr(batch, "row_tenant", None)
            ten = (torch.as_tensor(rt[:ft0].astype(np.int64), device=self.dev)
                   if self.ex.lora_rank and rt is not None and rt.size else None)
            for l in range(c.n_layers):
                x = self.model.layer(l, x, pos, attend, tenant=ten)
            if batch.n_dec:
                logits = self.model.final(x[batch.dec_rows.tolist()]).cpu()
        # teacher forcing: the next decode input of each slot is the GPU's greedy token
        for slot, tok in zip(batch.dec_slots.tolist(), gpu_tokens):
            self.last_token[slot] = int(tok)
        # post-tick per-head trims (the reference's kept[h] after Engine._exec_decode)
        for slot, kept in kept_post.items():
            d = self.dec[slot]
            end = len(d["k"][0])
            d["first"] = [max(f, end - kk) for f, kk in zip(d["first"], kept)]
        ft = None
        if batch.ft_pairs:
            pairs = [(p.rid, p.prompt, p.chosen, p.rejected, getattr(p, "tenant", 0)) for p in batch.ft_pairs]
            losses, margins, grads = self.ex.dpo_step(pairs, coef_margins=ft_margins)
            grads = {n: g.cpu() for n, g in grads.items()}
            self.ex.adamw({n: g.to(self.dev) for n, g in grads.items()}, tenants=[p[4] for p in pairs])
            ft = (losses, margins, grads)
        return logits, ft
