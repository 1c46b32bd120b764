"""HybridModel: executes one hybrid tick (prefill + decode + DPO fine-tune rows in ONE ragged batch)
entirely through libmace_b200.so.

This is what replaces the cost-model charge inside the reference's Engine._execute
(engine.py:573-676): the reference *charges* max(member latency) for a bin and moves MB counters; here
the bin's rows run through the decoder layers, decode rows emit greedy tokens, and fine-tune rows
produce the DPO loss and a masked AdamW update of the selected layers.

torch is used only for device memory, streams and memcpy/memset; every arithmetic op is a launch of a
hand-written sm_100a kernel (see csrc/). Device state that persists across ticks:
  weights (bf16), fp32 master/m/v/grad of the selected parameters, frozen pi_ref copies,
  head-major KV page pools + page tables + the decode-page free stack, last greedy token per slot.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import (Ctx, MaceKvLayout, MaceLayerGrads, MaceLayerWeights, MaceLoraLayer, MaceModelDesc, MaceSavedActs,
                   MaceTickBuffers, MaceTickDesc)
from .batch import PAGE, TickBatch
from .config import (LORA_PROJ, ModelConfig, TrainConfig, selected_param_names, sensitivity_ranking,
                     trainable_param_names)
from .kvmanager import DecodePageMirror
from .weights import init_lora


@dataclass
class StepOutputs:
    dec_tokens: torch.Tensor | None     # [n_dec] int32 (device)
    ft_loss: torch.Tensor | None        # [n_pairs] fp32
    ft_margin: torch.Tensor | None
    ft_lp: torch.Tensor | None          # [n_pairs, 2] policy log-probs
    ref_lp: torch.Tensor | None         # [n_pairs, 2] pi_ref log-probs used
    head_norm: torch.Tensor | None      # [n_dec, Hq] per-head attention-output norms of the last layer


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class HybridModel:
    def __init__(
        self,
        cfg: ModelConfig,
        tcfg: TrainConfig,
        weights: dict[str, torch.Tensor],
        *,
        device: int = 0,
        max_slots: int = 1024,
        max_prompt_len: int = 4096,
        max_decode_steps: int = 512,
        prompt_groups: int = 4096,
        decode_pages: int | None = None,
        ctx: Ctx | None = None,
        process_group=None,
        grad_allreduce: str = "bf16",
        n_tenants: int = 1,
        lora_weights: dict[str, torch.Tensor] | None = None,
        lora_seed: int = 0,
    ):
        self.cfg, self.tcfg = cfg, tcfg
        self.ctx = ctx or Ctx(device)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.current_stream(self.dev)
        self.pg = process_group
        self.grad_allreduce = grad_allreduce
        d, L = cfg.d_model, cfg.n_layers
        self.w = {n: t.to(self.dev, torch.bfloat16).contiguous() for n, t in weights.items()}
        # the masked AdamW rewrites the selected parameters' bf16 working copies in place: never alias the caller's
        # tensors (a bf16 dict already on this device would otherwise be trained under the caller's feet)
        for n in selected_param_names(cfg, tcfg):
            if self.w[n].data_ptr() == weights[n].data_ptr():
                self.w[n] = self.w[n].clone()
        # ---- per-tenant LoRA adapters (TrainConfig.lora_rank): the selected layers' projections carry them, the base
        # model is frozen and shared by every tenant
        self.lora = bool(tcfg.lora_rank)
        self.n_tenants = n_tenants
        self.lora_R = 0
        self.sel_layers = tcfg.selected_layers(cfg)
        if self.lora:
            if tcfg.sensitivity_topk is not None:
                raise ValueError("LoRA adapters and sensitivity-selected layers are exclusive")
            self.lora_R = n_tenants * tcfg.lora_rank
            if self.lora_R % 8:
                raise ValueError("LoRA: tenants x rank must be a multiple of 8")
            lw = lora_weights if lora_weights is not None else init_lora(cfg, tcfg, n_tenants, lora_seed)
            self.lora_init = {n: t.float().cpu().clone() for n, t in lw.items()}
            self._build_lora(lw)
        # ---- trainable parameters: flat fp32 master / m / v / grad + segment table for masked AdamW
        self.sel = trainable_param_names(cfg, tcfg, n_tenants)
        self.l_min = min(self.sel_layers)
        src = self.lw if self.lora else self.w
        sizes = [src[n].numel() for n in self.sel]
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.n_sel = int(offs[-1])
        self.master = torch.cat([src[n].float().reshape(-1) for n in self.sel])
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.grad = torch.zeros_like(self.master)
        self._g16 = torch.empty(self.n_sel, dtype=torch.bfloat16, device=self.dev) if process_group is not None else None
        self.gview = {n: self.grad[offs[i]: offs[i + 1]].view(src[n].shape) for i, n in enumerate(self.sel)}
        self.seg_offsets = torch.from_numpy(offs).to(self.dev)
        self.seg_ptrs = torch.tensor([src[n].data_ptr() for n in self.sel], dtype=torch.int64, device=self.dev)
        self.adam_step = 0
        self.update_layers: list[int] | None = None  # sensitivity selection (TrainConfig.sensitivity_topk)
        self.update_names = list(self.sel)
        self.sensitivity: list | None = None
        # the float4 AdamW kernel needs every segment to start on a 4-element boundary of the flat buffers and
        # every bf16 working copy 8-byte aligned (true for every preset: all widths are multiples of 4)
        self.adam_vec4 = bool((offs % 4 == 0).all() and all(src[n].data_ptr() % 8 == 0 for n in self.sel))
        # pi_ref frozen at init; with LoRA the frozen base IS pi_ref (adapters masked off)
        self.ref_w = {} if self.lora else {n: self.w[n].clone() for n in self.sel}
        if self.lora:
            self._build_tenant_segments(offs)
        # pi_ref log-probs are recomputed in every fine-tune tick by default: the pi_ref and policy sub-passes then
        # start from the SAME tick's layer-l_min activations, so the bf16 noise of the rows below l_min cancels in
        # the margin (lp - ref). A pi_ref cached from the pair's first tick was computed inside a different batch
        # (other tile shapes / accumulation orders below l_min) and left ~0.1 nat of noise in m on later steps.
        # The cost is one sub-pass over the selected layers only; most ticks need it anyway (a new pair).
        self.ref_every_tick = True
        # ---- RoPE tables (fp64 on host -> fp32)
        half = cfg.head_dim // 2
        inv = cfg.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim)
        # RoPE is computed, not learned: the table covers every position a request of this model can reach
        # (GPT-2's learned table is bounded by cfg.max_pos; GpuEngine.build_batch refuses positions past it)
        n_pos = max(cfg.max_pos, max_prompt_len + max_decode_steps)
        ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
        self.cos_t = torch.from_numpy(np.cos(ang).astype(np.float32)).to(self.dev)
        self.sin_t = torch.from_numpy(np.sin(ang).astype(np.float32)).to(self.dev)
        # ---- KV pools and page tables
        H, hd = cfg.n_kv_heads, cfg.head_dim
        self.max_slots = max_slots
        self.maxpp = (max_prompt_len + PAGE - 1) // PAGE
        self.maxdp = (max_decode_steps + PAGE - 1) // PAGE + 2
        self.prompt_groups = prompt_groups
        if decode_pages is None:
            decode_pages = max_slots * H * 4
        self.max_prompt_len = max_prompt_len
        self.decode_pages = decode_pages
        # + 1: the reserved sink page (kvpage.cu) an exhausted pop would point at -- never on the free stack
        self.pages_per_layer = prompt_groups * H + decode_pages + 1
        # zero-initialised: page rows outside a sequence's window are multiplied by exact zeros on the
        # tensor cores, so they must hold finite values
        self.k_pool = torch.zeros(L, self.pages_per_layer, PAGE, hd, dtype=torch.bfloat16, device=self.dev)
        self.v_pool = torch.zeros_like(self.k_pool)
        i32 = dict(dtype=torch.int32, device=self.dev)
        self.ptab = torch.zeros(max_slots, self.maxpp, **i32)
        self.dtab = torch.zeros(max_slots, H, self.maxdp, **i32)
        self.dec_base = torch.zeros(max_slots, H, **i32)
        self.dec_first = torch.zeros(max_slots, H, **i32)
        self.dec_end = torch.zeros(max_slots, **i32)
        self.free_stack = torch.arange(prompt_groups * H, self.pages_per_layer - 1, **i32)
        self.free_top = torch.tensor([decode_pages, 0], **i32)  # {stack top, status}
        self.kv_mirror = DecodePageMirror(max_slots, H, decode_pages)  # host count of the same pops / pushes
        # decode-window compaction (mace_kv_compact): on demand when a tick's page pops exceed the free pages, and
        # after every prune trim for windows of <= compact_max_window tokens (0: off -- a window slides one slot per
        # tick, so its straddled leading page empties by itself within < 16 ticks; re-basing it every tick would
        # move the window each tick for at most one page); bytes moved / pages returned
        self.compact_max_window = int(os.environ.get("MACE_KV_COMPACT_MAX", "0"))
        self.compaction_bytes = 0
        self.compaction_pages = 0
        self.last_token = torch.zeros(max_slots, **i32)
        self.dec_counters = torch.zeros(max_slots * H, **i32)  # decode chunk-merge counters (self-cleaning)
        # decode ticket counter: zero between launches -- the warp that draws a launch's terminal ticket resets
        # it, which needs every launched warp to enter the ticket loop (launch_decode2: base == grid * WARPS)
        self.dec_work = torch.zeros(1, dtype=torch.int64, device=self.dev)
        # 0 auto (tcgen05 swap-AB for GQA, CUDA-core streaming for MHA), 1 / 2 forced (MACE_DECODE_IMPL: sweeps)
        self.decode_impl = int(os.environ.get("MACE_DECODE_IMPL", "0"))
        # prefill / FT attention as query-block PAIRS (two 128-row tiles per CTA, csrc/attention_fa2.cu) for head_dim
        # 64 / 128; MACE_ATTN_PAIRS=0 keeps the single-tile kernel (A/B). The engine builds the tile items to match.
        self.attn_pairs = cfg.head_dim in (64, 128) and os.environ.get("MACE_ATTN_PAIRS", "1") != "0"
        self.kv = MaceKvLayout(
            ptab=self.ptab.data_ptr(), max_prompt_pages=self.maxpp, dtab=self.dtab.data_ptr(),
            max_dec_pages=self.maxdp, dec_base=self.dec_base.data_ptr(), dec_first=self.dec_first.data_ptr(),
            dec_end=self.dec_end.data_ptr(), free_stack=self.free_stack.data_ptr(),
            free_top=self.free_top.data_ptr(), stack_cap=decode_pages, n_kv_heads=H,
            sink_page=self.pages_per_layer - 1,
        )
        self._cap = 0
        self._ft_cap = 0
        self._R_cap = 0
        self._ndec_cap = 0
        self._P_cap = 0
        # padded vocab row stride (16-byte aligned fp32/bf16 rows: TMA operand / TMA-store epilogue)
        self.vpad = (cfg.vocab + 7) // 8 * 8
        self.ws = torch.empty(16 << 20, dtype=torch.float32, device=self.dev)  # 64 MB split-K / reduction scratch
        self.tape: list | None = None   # when a list: every device-side call is appended (bench replay)
        self._stage_ring: list = [(None, None)] * 8   # pinned staging buffers (+ the event of their last copy)
        self._stage_dev: list = [None] * 8             # device scratch per staging slot
        self._stage_i = 0
        self.instrument: list | None = None  # when a list: (ev0, ev1, bytes) per decode-attention launch
        self.gemm_instrument: list | None = None  # when a list: (ms, flops, launches) of the GEMMs of each tick
        self._attn_bytes = 0
        self.idx = torch.empty(1 << 16, dtype=torch.int32, device=self.dev)
        self._bufs = MaceTickBuffers()
        # True: the decode head writes the fp32 logits [n_dec, V] and takes the argmax over them (recorded oracle
        # replays read the logits); False: the lm_head GEMM's epilogue reduces each row to its argmax directly
        self.keep_dec_logits = os.environ.get("MACE_DEC_LOGITS") == "1"  # A/B switch
        self.mh = self._create_native()

    def _build_lora(self, lw: dict[str, torch.Tensor]) -> None:
        """Device layout of the adapters (include/mace_b200.h MaceLoraLayer):
          qkv / up   augmented base weight [out, d + R] = [W | B]: the forward [h | Zm] . [W | B]^T is one GEMM
          o / down   A stacked under the base weight [d + R, in] = [W; A]: the backward [dY | dZ] . [W; A] is one GEMM
        Every adapter also has a contiguous bf16 working copy per name (self.lw: AdamW's per-tenant targets); for
        a_o / a_down that copy IS the stacked block, for bt_qkv / bt_up it is scattered into the augmented weight
        after each update (mace_lora_bt_scatter)."""
        c, dev, R = self.cfg, self.dev, self.lora_R
        D = c.d_model
        bf = dict(dtype=torch.bfloat16, device=dev)
        self.lw: dict[str, torch.Tensor] = {}
        for l in self.sel_layers:
            p, q = f"layers.{l}.", f"lora.{l}."
            for proj in ("qkv", "up"):
                W = self.w[p + proj + ".w"]
                aug = torch.empty(W.shape[0], D + R, **bf)
                aug[:, :D] = W
                bt = lw[q + "bt_" + proj].to(dev, torch.bfloat16).contiguous()
                aug[:, D:] = bt.t()
                self.w[p + proj + ".w"] = aug
                self.lw[q + "a_" + proj] = lw[q + "a_" + proj].to(dev, torch.bfloat16).contiguous()
                self.lw[q + "bt_" + proj] = bt
            for proj in ("o", "down"):
                W = self.w[p + proj + ".w"]
                st = torch.empty(D + R, W.shape[1], **bf)
                st[:D] = W
                st[D:] = lw[q + "a_" + proj].to(dev, torch.bfloat16)
                self.w[p + proj + ".w"] = st
                self.lw[q + "a_" + proj] = st[D:]
                self.lw[q + "bt_" + proj] = lw[q + "bt_" + proj].to(dev, torch.bfloat16).contiguous()
        self.tenant_steps = np.zeros(self.n_tenants, np.int64)
        self._tick_tenants: list[int] = []

    def _build_tenant_segments(self, offs: np.ndarray) -> None:
        """Per tenant u, the AdamW segment table of its adapter rows: for every adapter tensor [R, width] the rows
        [u * rank, (u + 1) * rank) -- one contiguous run of rank * width elements in the flat buffers and in the bf16
        working copy."""
        r = self.tcfg.lora_rank
        self._tenant_seg = []
        for u in range(self.n_tenants):
            vstart, flat, wp = [0], [], []
            for i, n in enumerate(self.sel):
                k = r * self.lw[n].shape[1]
                flat.append(int(offs[i]) + u * k)
                wp.append(self.lw[n].data_ptr() + 2 * u * k)
                vstart.append(vstart[-1] + k)
            dev64 = lambda a: torch.tensor(a, dtype=torch.int64, device=self.dev)  # noqa: E731
            self._tenant_seg.append((dev64(vstart), dev64(flat), dev64(wp), vstart[-1]))

    def _create_native(self):
        """mace_model_create: weight / gradient / KV pointers of the native tick executor (csrc/tick.cu)."""
        c = self.cfg
        w = self.w
        fields = [f for f, _ in MaceLayerWeights._fields_]

        def lw(get, l, cls):
            return cls(**{f: get(f"layers.{l}.{f[:-2]}.{f[-1]}") for f in fields})

        def wptr(n):
            t = w.get(n)
            return None if t is None else t.data_ptr()

        def refptr(n):
            t = self.ref_w.get(n, w.get(n))
            return None if t is None else t.data_ptr()

        def gptr(n):
            t = self.gview.get(n)
            return None if t is None else t.data_ptr()

        L = c.n_layers
        self._layers_arr = (MaceLayerWeights * L)(*[lw(wptr, l, MaceLayerWeights) for l in range(L)])
        nsel = len(self.sel_layers)
        self._sel_arr = (C.c_int * max(nsel, 1))(*self.sel_layers)
        self._ref_arr = (MaceLayerWeights * max(nsel, 1))(*[lw(refptr, l, MaceLayerWeights) for l in self.sel_layers])
        self._grad_arr = (MaceLayerGrads * max(nsel, 1))(*[lw(gptr, l, MaceLayerGrads) for l in self.sel_layers])
        desc = MaceModelDesc(
            family=int(c.family == "gpt2"), n_layers=L, d_model=c.d_model, n_heads=c.n_heads,
            n_kv_heads=c.n_kv_heads, head_dim=c.head_dim, ffn=c.ffn, up_dim=c.up_dim, vocab=c.vocab,
            norm_eps=c.norm_eps, dpo_beta=self.tcfg.dpo_beta,
            embed=wptr("embed"), pos_embed=wptr("pos_embed"), final_norm_w=wptr("final_norm.w"),
            final_norm_b=wptr("final_norm.b"), layers=self._layers_arr, n_sel=nsel, sel_layers=self._sel_arr,
            ref_layers=self._ref_arr, ref_final_norm_w=refptr("final_norm.w"), ref_final_norm_b=refptr("final_norm.b"),
            grads=self._grad_arr, grad_final_norm_w=gptr("final_norm.w"), grad_final_norm_b=gptr("final_norm.b"),
            grad_flat=self.grad.data_ptr(), n_grad=self.n_sel, cos_t=self.cos_t.data_ptr(),
            sin_t=self.sin_t.data_ptr(), kv=self.kv, k_pool=self.k_pool.data_ptr(), v_pool=self.v_pool.data_ptr(),
            pages_per_layer=self.pages_per_layer, last_token=self.last_token.data_ptr(),
            dec_counters=self.dec_counters.data_ptr(), dec_work=self.dec_work.data_ptr(),
            decode_impl=int(self.decode_impl), attn_pairs=int(self.attn_pairs),
        )
        if self.lora:
            def lptr(l, n):
                return self.lw[f"lora.{l}.{n}"].data_ptr()

            def lgrad(l, n):
                return self.gview[f"lora.{l}.{n}"].data_ptr()

            self._lora_arr = (MaceLoraLayer * nsel)(*[MaceLoraLayer(
                **{f"a_{p}": lptr(l, f"a_{p}") for p in LORA_PROJ},
                bt_o=lptr(l, "bt_o"), bt_down=lptr(l, "bt_down"),
                **{f"g_a_{p}": lgrad(l, f"a_{p}") for p in LORA_PROJ},
                **{f"g_bt_{p}": lgrad(l, f"bt_{p}") for p in LORA_PROJ}) for l in self.sel_layers])
            desc.lora_R, desc.lora_rank, desc.lora_scale = self.lora_R, self.tcfg.lora_rank, self.tcfg.lora_scale
            desc.lora = self._lora_arr
        h = C.c_void_p()
        self.ctx.check(self.ctx.L.mace_model_create(self.ctx.h, C.byref(desc), C.byref(h)), "mace_model_create")
        return h

    def set_decode_impl(self, impl: int) -> None:
        """0 auto, 1 CUDA-core streaming decode attention, 2 tcgen05 swap-AB (re-creates the executor)."""
        self.decode_impl = impl
        self.ctx.L.mace_model_destroy(self.mh)
        self.mh = self._create_native()

    def __del__(self):
        try:
            if getattr(self, "mh", None):
                self.ctx.L.mace_model_destroy(self.mh)
                self.mh = None
        except Exception:
            pass

    def ft_bytes_per_token(self) -> int:
        """Device bytes one fine-tune token occupies (the per-row buffers _ensure sizes for FT rows: saved
        activations of every selected layer + the pi_ref / backward scratch). This is what the reference's
        ft_mem_per_token (cost_model.py:40-41) stands for on a B200 (C5 sizes the cost model with it)."""
        c = self.cfg
        qo = c.n_heads * c.head_dim
        sav = 4 * c.d_model + 2 * c.d_model + 2 * c.qkv_dim + 2 * qo + 4 * c.n_heads + 4 * c.d_model + 2 * c.d_model \
            + 2 * c.up_dim + 2 * c.ffn
        scratch = (3 * 4 * c.d_model + 4 * c.n_heads + 2 * c.d_model + 2 * c.qkv_dim + 2 * qo + 2 * c.up_dim + 2 * c.ffn
                   + 4 * c.d_model + 2 * c.d_model + 4 * max(c.ffn, c.up_dim, c.qkv_dim, qo) + 2 * c.ffn + 2 * c.up_dim
                   + 2 * qo + 4 * c.qkv_dim + 2 * c.qkv_dim)
        return len(self.sel_layers) * sav + scratch

    # ------------------------------------------------------------------ buffers
    def _ensure(self, T: int, n_ft: int, R: int, n_dec: int, P: int = 1) -> None:
        c, dev = self.cfg, self.dev
        grew = False
        bf, f32 = dict(dtype=torch.bfloat16, device=dev), dict(dtype=torch.float32, device=dev)
        LR = self.lora_R  # adapter columns (tenants x rank); R below is the tick's logit rows
        ldh = c.d_model + LR  # LoRA layers: [h | Zm] rows
        if T > self._cap:
            cap = max(T, int(self._cap * 1.5), 256)
            self.x = torch.empty(cap, c.d_model, **f32)
            self.h = torch.empty(cap, ldh, **bf)
            if LR:
                self.lz = torch.empty(cap, LR, **f32)
                self.lzm = torch.empty(cap, LR, **bf)
            self.qkv = torch.empty(cap, c.qkv_dim, **bf)
            self.o = torch.empty(cap, c.n_heads * c.head_dim, **bf)
            self.lse = torch.empty(cap, c.n_heads, **f32)
            self.hn = torch.empty(cap, c.n_heads, **f32)
            self.u = torch.empty(cap, c.up_dim, **bf)
            self.a = torch.empty(cap, c.ffn, **bf)
            self._cap = cap
            grew = True
        if n_ft > self._ft_cap:
            cap = max(n_ft, int(self._ft_cap * 1.5), 128)
            self.sav = {}
            for l in self.sel_layers:
                self.sav[l] = dict(
                    x_in=torch.empty(cap, c.d_model, **f32), h1=torch.empty(cap, ldh, **bf),
                    qkv=torch.empty(cap, c.qkv_dim, **bf), o=torch.empty(cap, c.n_heads * c.head_dim, **bf),
                    lse=torch.empty(cap, c.n_heads, **f32), x_mid=torch.empty(cap, c.d_model, **f32),
                    h2=torch.empty(cap, ldh, **bf), u=torch.empty(cap, c.up_dim, **bf),
                    a=torch.empty(cap, c.ffn, **bf),
                )
                if LR:
                    self.sav[l].update(zm_o=torch.empty(cap, LR, **bf), zm_d=torch.empty(cap, LR, **bf))
            # ref-pass + backward scratch (FT rows only)
            self.rx = torch.empty(cap, c.d_model, **f32)
            self.rx2 = torch.empty(cap, c.d_model, **f32)
            self.x_lmin = torch.empty(cap, c.d_model, **f32)
            self.rlse = torch.empty(cap, c.n_heads, **f32)
            self.rh = torch.empty(cap, ldh, **bf)
            self.rqkv = torch.empty(cap, c.qkv_dim, **bf)
            self.ro = torch.empty(cap, c.n_heads * c.head_dim, **bf)
            self.ru = torch.empty(cap, c.up_dim, **bf)
            self.ra = torch.empty(cap, c.ffn, **bf)
            self.dx = torch.empty(cap, c.d_model, **f32)
            self.dy16 = torch.empty(cap, ldh, **bf)
            self.df = torch.empty(cap, max(c.ffn, c.up_dim, c.qkv_dim, c.n_heads * c.head_dim, ldh), **f32)
            if LR:
                self.ldz = torch.empty(cap, LR, **bf)
            self.da16 = torch.empty(cap, c.ffn, **bf)
            self.du16 = torch.empty(cap, c.up_dim, **bf)
            self.do16 = torch.empty(cap, c.n_heads * c.head_dim, **bf)
            self.dqkv = torch.empty(cap, c.qkv_dim, **f32)
            self.dqkv16 = torch.empty(cap, c.qkv_dim, **bf)
            self.Dbuf = torch.empty(cap, c.n_heads, **f32)
            # deterministic dQ order counters of the attention backward (left zeroed by every launch): the key blocks'
            # dQ contributions are added in a fixed order, so every fine-tune step is bitwise reproducible; about
            # 2.5x the backward kernel's time (0.2% of a C4 tick -> 0.5%). MACE_DQ_ATOMIC=1: fp32 atomics instead
            self.dq_order = torch.zeros(cap * c.n_heads, dtype=torch.int32, device=dev)
            self._ft_cap = cap
            grew = True
        if R > self._R_cap:
            cap = max(R, int(self._R_cap * 1.5), 64)
            self.ft_h = torch.empty(cap, c.d_model, **bf)
            self.ft_logits = torch.empty(cap, self.vpad, **f32)
            self.dlogits = torch.empty(cap, self.vpad, **bf)
            self.dh = torch.empty(cap, c.d_model, **f32)
            self.row_lse = torch.empty(cap, **f32)
            self.row_lp = torch.empty(cap, **f32)
            self._R_cap = cap
            grew = True
        if n_dec > self._ndec_cap:
            cap = max(n_dec, int(self._ndec_cap * 1.5), 64)
            self.dec_h = torch.empty(cap, c.d_model, **bf)
            self.dec_logits = torch.empty(cap, self.vpad, **f32)
            self.dec_tok = torch.empty(cap, dtype=torch.int32, device=dev)
            self.dec_keys = torch.zeros(cap, dtype=torch.int64, device=dev)  # fused argmax keys (self-cleaning)
            self.dec_ws = torch.empty(cap * c.n_kv_heads * 4 * (2 * c.group + c.group * c.head_dim), **f32)
            self._ndec_cap = cap
            grew = True
        if P > self._P_cap:
            cap = max(P, 2 * self._P_cap, 16)
            self.dpo_lp = torch.empty(cap, 2, **f32)
            self.dpo_ref_lp = torch.empty(cap, 2, **f32)
            self.dpo_loss = torch.empty(cap, **f32)
            self.dpo_margin = torch.empty(cap, **f32)
            self.dpo_coef = torch.empty(cap, 2, **f32)
            self._P_cap = cap
            grew = True
        if grew:
            self._fill_bufs()

    def _fill_bufs(self) -> None:
        """(Re)point the native executor's MaceTickBuffers at the current scratch tensors."""
        b = MaceTickBuffers()
        for n in ("x", "h", "qkv", "o", "lse", "hn", "u", "a"):
            setattr(b, n, getattr(self, n).data_ptr())
        b.ld_h = self.cfg.d_model + self.lora_R
        if self.lora:
            b.lz, b.lzm = self.lz.data_ptr(), self.lzm.data_ptr()
            if self._ft_cap:
                b.ldz = self.ldz.data_ptr()
        if self._ft_cap:
            sav = [MaceSavedActs(**{k: t.data_ptr() for k, t in self.sav[l].items()}) for l in self.sel_layers]
            self._sav_arr = (MaceSavedActs * max(len(sav), 1))(*sav)
            b.sav = self._sav_arr
            for n in ("rx", "rx2", "x_lmin", "rlse", "rh", "rqkv", "ro", "ru", "ra", "dx", "dy16", "df", "da16",
                      "du16", "do16", "dqkv", "dqkv16", "Dbuf", "dq_order"):
                setattr(b, n, getattr(self, n).data_ptr())
            if os.environ.get("MACE_DQ_ATOMIC") == "1":
                b.dq_order = None
            b.ld_df = self.df.shape[1]
        if self._R_cap:
            for n in ("ft_h", "ft_logits", "dlogits", "dh", "row_lse", "row_lp"):
                setattr(b, n, getattr(self, n).data_ptr())
            b.ld_vocab = self.vpad
        b.ld_vocab = self.vpad
        if self._ndec_cap:
            for n in ("dec_h", "dec_logits", "dec_tok", "dec_ws"):
                setattr(b, n, getattr(self, n).data_ptr())
            b.dec_ws_bytes = self.dec_ws.numel() * 4
            b.dec_keys = self.dec_keys.data_ptr()
        if self._P_cap:
            b.lp, b.ref_lp, b.loss = self.dpo_lp.data_ptr(), self.dpo_ref_lp.data_ptr(), self.dpo_loss.data_ptr()
            b.margin, b.coef = self.dpo_margin.data_ptr(), self.dpo_coef.data_ptr()
        b.ws, b.ws_bytes = self.ws.data_ptr(), self.ws.numel() * 4
        self._bufs = b

    def replay(self, tape) -> None:
        """Re-issue a recorded sequence of device calls (bench: device-only throughput)."""
        for op in tape:
            if op[0] == "step":
                self.step(op[1], ft_global=op[2])
            elif op[0] == "trim":
                self.apply_trim(op[1], op[2])
            elif op[0] == "idle_update":
                self.idle_update()
            else:
                self.release_slots(op[1])

    @staticmethod
    def tape_collectives(tape) -> int:
        """Gradient all-reduces a tape issues (equal on every rank of a lockstep run)."""
        return sum(1 for op in tape if op[0] == "idle_update" or (op[0] == "step" and (
            op[2] or (op[1].ft_pairs and op[1].T > op[1].ft0))))

    def _upload(self, batch: TickBatch) -> dict[str, int | None]:
        if getattr(batch, "_packed", None) is None:
            batch._packed = batch.packed()
        buf, layout = batch._packed
        n = buf.size
        if n > self.idx.numel():
            self.idx = torch.empty(int(n * 1.5), dtype=torch.int32, device=self.dev)
        # a fresh block from torch's caching pinned allocator per tick: the allocator records the copy's
        # stream event, so the host can run ticks ahead without overwriting an in-flight H2D source
        host = torch.from_numpy(buf).pin_memory()
        self.idx[:n].copy_(host, non_blocking=True)
        self.h2d_bytes = n * 4
        # device addresses of the packed tables (int32 each; None for an empty table)
        base = self.idx.data_ptr()
        return {name: (base + 4 * off if (len(shape) and math.prod(shape)) else None)
                for name, (off, shape) in layout.items()}

    # ------------------------------------------------------------------ tick
    @torch.no_grad()
    def step(self, batch: TickBatch, trim: tuple[np.ndarray, np.ndarray] | None = None,
             ft_global: bool | None = None) -> StepOutputs:
        """Run one hybrid tick on the device (asynchronous; outputs are device tensors).

        Every launch of the tick is issued by ONE native call (mace_tick_run, csrc/tick.cu); this
        method only sizes the buffers, uploads the packed row tables and fills the descriptor.
        ``ft_global``: whether ANY replica has fine-tune rows this tick (lockstep multi-GPU); defaults to
        this replica's own rows."""
        if self.tape is not None:
            self.tape.append(("step", batch, ft_global))
        T, ft0 = batch.T, batch.ft0
        n_ft = T - ft0
        R = int(batch.ft_logit_rows.shape[0])
        n_dec = batch.n_dec
        P = len(batch.ft_pairs)
        self._ensure(max(T, 1), max(n_ft, 1), max(R, 1), max(n_dec, 1), max(P, 1))
        if n_dec:  # raises KvCapacityError before any launch if the decode pages cannot hold this tick
            ds = batch.dec_slots.astype(np.int64)
            if self.kv_mirror.pops(ds) > self.kv_mirror.free:  # memory pressure: reclaim straddled pages first
                self.compact_windows()
            self.kv_mirror.alloc(ds)
        v = self._upload(batch)
        has_ft = n_ft > 0 and P > 0
        if self.instrument is not None and n_dec:
            self._attn_bytes = self.decode_attn_bytes(batch)
        d = MaceTickDesc(T=T, ft0=ft0, n_dec=n_dec, R=R, n_pairs=P,
                         need_ref=int(self.ref_every_tick or any(p.ref_lp is None for p in batch.ft_pairs)))
        for name in ("tokens", "pos", "row_seq", "row_kvi", "seqs", "dec_slots", "dec_rows", "ptab_slots",
                     "ptab_rows", "page_copies", "ft_local_rows", "ft_targets", "pair_rows", "row_ps", "ref_cached",
                     "ft_seqs", "ft_row_seq"):
            setattr(d, name, v[name])
        d.tc_items, d.n_tc = v["tc_items"], batch.tc_items.shape[0]
        d.n_tc_inference = int(batch.meta.get("n_tc_inference", d.n_tc))
        d.dec_items, d.n_dec_items = v["dec_items"], batch.dec_items.shape[0]
        d.n_ptab, d.ptab_cols = batch.ptab_slots.shape[0], batch.ptab_rows.shape[1] if batch.ptab_rows.ndim == 2 else 0
        d.n_copies = batch.page_copies.shape[0]
        d.ft_tc_items, d.n_ft_tc = v["ft_tc_items"], batch.ft_tc_items.shape[0]
        d.bwd_items, d.n_bwd = v["bwd_items"], batch.bwd_items.shape[0]
        if self.lora:
            if batch.row_tenant.shape[0] != T or (T and int(batch.row_tenant.max()) >= self.n_tenants):
                raise ValueError(f"LoRA tick needs a tenant per row, each < {self.n_tenants}")
            d.row_tenant = v["row_tenant"]
            self._tick_tenants = sorted({p.tenant for p in batch.ft_pairs}) if has_ft else []
        events = None
        if self.instrument is not None and n_dec and T:
            events = [torch.cuda.Event(enable_timing=True) for _ in range(2 * self.cfg.n_layers)]
            for e in events:
                e.record()  # materialise the cudaEvent_t handles
            arr = (C.c_void_p * len(events))(*[e.cuda_event for e in events])
            d.attn_events = C.cast(arr, C.c_void_p)
            self._ev_keep = arr
        gcount = None
        if self.gemm_instrument is not None:  # CUDA events around every GEMM of the tick (bench roofline pass)
            cap = 4096
            if getattr(self, "_gev", None) is None:
                self._gev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * cap)]
                for e in self._gev:
                    e.record()
                self._gev_arr = (C.c_void_p * (2 * cap))(*[e.cuda_event for e in self._gev])
                self._gflops = np.zeros(cap, np.int64)
            gcount = np.zeros(1, np.int32)
            d.gemm_events, d.gemm_events_cap = C.cast(self._gev_arr, C.c_void_p), cap
            d.gemm_flops, d.gemm_count = self._gflops.ctypes.data, gcount.ctypes.data
        if self._ndec_cap:  # fused lm_head argmax unless the caller reads the decode logits (oracle replays)
            self._bufs.dec_keys = None if self.keep_dec_logits else self.dec_keys.data_ptr()
        self.ctx.check(self.ctx.L.mace_tick_run(self.mh, C.byref(self._bufs), C.byref(d), self._s), "mace_tick_run")
        if gcount is not None:
            torch.cuda.synchronize(self.dev)
            n = int(gcount[0])
            ms = sum(self._gev[2 * i].elapsed_time(self._gev[2 * i + 1]) for i in range(n))
            self.gemm_instrument.append((ms, int(self._gflops[:n].sum()), n))
        if events is not None:
            for l in range(self.cfg.n_layers):
                self.instrument.append((events[2 * l], events[2 * l + 1], self._attn_bytes))
        out = StepOutputs(None, None, None, None, None, None)
        if n_dec and T:
            out.dec_tokens = self.dec_tok[:n_dec]
            d0 = int(batch.dec_rows[0])  # decode rows are contiguous in the batch (engine.build_batch)
            out.head_norm = self.hn[d0: d0 + n_dec]  # ||o_{t,h}|| of the last layer's attention, per query head
        if trim is not None and trim[0].size:
            self.apply_trim(*trim)
        if has_ft:
            out.ft_loss, out.ft_margin = self.dpo_loss[:P], self.dpo_margin[:P]
            out.ft_lp, out.ref_lp = self.dpo_lp[:P], self.dpo_ref_lp[:P]
        if has_ft or ft_global:
            self.apply_update(has_ft)
        return out

    @property
    def _s(self) -> int:
        return torch.cuda.current_stream(self.dev).cuda_stream

    def _chk(self, rc, what):
        self.ctx.check(rc, what)

    def kv_status(self) -> tuple[int, int]:
        """(device free-stack top, status word) -- synchronous; status != 0 means a pop found the stack
        empty, which the host mirror makes unreachable (tests assert the top equals the mirror's count)."""
        out = (C.c_int * 2)()
        self.ctx.check(self.ctx.L.mace_kv_status(self.ctx.h, C.byref(self.kv), out), "kv_status")
        return int(out[0]), int(out[1])

    def decode_attn_bytes(self, batch: TickBatch) -> int:
        """Algorithmic bytes of ONE decode-attention launch (one layer) of this tick: every visible K and
        V row of every (decode sequence, kv head) read once + q rows read + o rows written (syncs)."""
        c = self.cfg
        slots = torch.from_numpy(batch.dec_slots.astype(np.int64)).to(self.dev)
        de = self.dec_end[slots].cpu().numpy()
        df = self.dec_first[slots].cpu().numpy()
        n_pv = batch.seqs[batch.seqs[:, 0] == 1][:, 4]
        tokens = int((n_pv[:, None] + (de[:, None] - df)).sum())
        return tokens * c.head_dim * 2 * 2 + batch.n_dec * c.n_heads * c.head_dim * 2 * 2

    def apply_trim(self, slots: np.ndarray, kept: np.ndarray) -> None:
        """Post-tick per-head prune trim (engine.py:506-529 decisions) -> page compaction on device."""
        n = slots.shape[0]
        if n == 0:
            return
        if self.tape is not None:
            self.tape.append(("trim", slots.copy(), kept.copy()))
        sl = np.asarray(slots, np.int64)
        self.kv_mirror.trim(sl, np.asarray(kept, np.int64).reshape(n, -1))
        dev = self._stage((np.ascontiguousarray(slots, np.int32).reshape(-1),
                           np.ascontiguousarray(kept, np.int32).reshape(-1)))
        self._chk(self.ctx.L.mace_kv_trim(self.ctx.h, C.byref(self.kv), dev, dev + 4 * n, n, self._s), "kv_trim")
        if self.compact_max_window:
            self.compact_windows(sl, self.compact_max_window)

    def compact_windows(self, slots: np.ndarray | None = None, max_w: int = 64) -> int:
        """Decode-window compaction (mace_kv_compact): every head of ``slots`` (default: every live slot) whose
        retained window of <= max_w tokens fits one page fewer when re-based at dec_first moves its K/V rows down
        inside its pages and returns the emptied page. Returns the pages reclaimed. Run on demand when a tick's
        page pops exceed the free pages (step), or after every trim with compact_max_window > 0."""
        if slots is None:
            slots = np.nonzero(self.kv_mirror.end > 0)[0]
        items = self.kv_mirror.compact(np.asarray(slots, np.int64), max_w)
        if not items.shape[0]:
            return 0
        c = self.cfg
        w = self.kv_mirror.end[items[:, 0]] - self.kv_mirror.first[items[:, 0], items[:, 1]]
        self.compaction_bytes += int(w.sum()) * c.n_layers * 2 * c.head_dim * 2 * 2  # read + write, K and V
        self.compaction_pages += int(items.shape[0])
        di = self._stage((items.reshape(-1),))
        self._chk(self.ctx.L.mace_kv_compact(self.ctx.h, C.byref(self.kv), di, items.shape[0], max_w, c.n_layers,
                                             c.head_dim, self.pages_per_layer, self.k_pool.data_ptr(),
                                             self.v_pool.data_ptr(), self._s), "kv_compact")
        return int(items.shape[0])

    def release_slots(self, slots: list[int]) -> None:
        if not slots:
            return
        if self.tape is not None:
            self.tape.append(("release", list(slots)))
        self.kv_mirror.release(np.asarray(slots, np.int64))
        dev = self._stage((np.asarray(slots, np.int32),))
        self._chk(self.ctx.L.mace_kv_release(self.ctx.h, C.byref(self.kv), dev, len(slots), self._s), "kv_release")

    def _stage(self, parts) -> int:
        """Copy small int32 host arrays (concatenated) to a device scratch buffer, stream-ordered, through a
        ring of pinned staging buffers; returns the device address. A staging buffer is reused only after
        the copy that last read it has completed (its event)."""
        n = sum(a.size for a in parts)
        ring = self._stage_ring
        i = self._stage_i = (self._stage_i + 1) % len(ring)
        host, ev = ring[i]
        if ev is not None:
            ev.synchronize()  # recorded many calls ago: normally already complete
        if host is None or host.numel() < n:
            host = torch.empty(max(n, 1 << 14), dtype=torch.int32, pin_memory=True)
        hv = host.numpy()
        o = 0
        for a in parts:
            hv[o: o + a.size] = a
            o += a.size
        if self._stage_dev[i] is None or self._stage_dev[i].numel() < n:
            self._stage_dev[i] = torch.empty(max(n, 1 << 14), dtype=torch.int32, device=self.dev)
        d = self._stage_dev[i]
        d[:n].copy_(host[:n], non_blocking=True)
        if ev is None:
            ev = torch.cuda.Event()
        ev.record()  # re-recorded only after its previous copy completed (synchronize above)
        ring[i] = (host, ev)
        return d.data_ptr()

    # ------------------------------------------------------------------ fine-tune update
    def _build_update_runs(self) -> None:
        """Contiguous runs of the flat optimizer buffers covering the updated parameters (the chosen layers + the
        final norm), each with its own device segment table: AdamW touches nothing else."""
        names = [n for n in self.sel if not n.startswith("layers.") or int(n.split(".")[1]) in self.update_layers]
        idx = {n: i for i, n in enumerate(self.sel)}
        offs = np.concatenate([[0], np.cumsum([self.w[n].numel() for n in self.sel])]).astype(np.int64)
        runs, cur = [], []
        for n in self.sel:
            if n in names:
                cur.append(n)
            elif cur:
                runs.append(cur)
                cur = []
        if cur:
            runs.append(cur)
        self._update_runs = []
        for run in runs:
            a = int(offs[idx[run[0]]])
            ro = np.array([offs[idx[n]] - a for n in run] + [offs[idx[run[-1]] + 1] - a], np.int64)
            self._update_runs.append((a, int(ro[-1]), torch.from_numpy(ro).to(self.dev),
                                      torch.tensor([self.w[n].data_ptr() for n in run], dtype=torch.int64,
                                                   device=self.dev), len(run)))
        self.update_names = names

    def idle_update(self) -> None:
        """A lockstep round this replica joins with a drained trace while another replica fine-tunes: zero
        gradients into the same all-reduce, then the same AdamW step (engine.run_ticks)."""
        if self.tape is not None:
            self.tape.append(("idle_update",))
        self.apply_update(False)

    def weight_checksum(self) -> int:
        """Order-independent 64-bit checksum of the fp32 master bits of the selected parameters (replicas must
        agree bit for bit; dist.Lockstep.assert_equal)."""
        bits = self.master.view(torch.int32).to(torch.int64)
        return int((bits * torch.arange(1, bits.numel() + 1, device=bits.device) % 1000003).sum().item())

    def apply_update(self, local_ft: bool) -> None:
        """Gradient exchange (NCCL all-reduce over the request-stream replicas) and the
        masked AdamW. A replica without FT rows this tick contributes zeros and applies the same
        update, so every replica keeps bit-identical weights. The exchange runs in bf16 by default
        (grad_allreduce "bf16": half the bytes, SURVEY §8(e)'s 872 MB at C4 top-2 layers): the fp32
        gradient is rounded once, summed by NCCL, and widened back before AdamW; "f32" keeps it exact."""
        L, s = self.ctx.L, self._s
        if not local_ft:
            self.grad.zero_()
        if self.lora:
            return self._apply_lora_update(local_ft)
        if self.pg is not None:
            if self.grad_allreduce == "bf16":
                g16 = self._g16
                self._chk(L.mace_f32_to_bf16(self.ctx.h, self.grad.data_ptr(), self.n_sel, g16.data_ptr(), s),
                          "grad to bf16")
                torch.distributed.all_reduce(g16, group=self.pg)
                self._chk(L.mace_bf16_to_f32(self.ctx.h, g16.data_ptr(), self.n_sel, self.grad.data_ptr(), s),
                          "grad to f32")
            else:
                torch.distributed.all_reduce(self.grad, group=self.pg)
        self.adam_step += 1
        t = self.tcfg
        if t.sensitivity_topk is not None:
            if self.update_layers is None:  # first update: rank the span by ||grad W_l|| / ||W_l|| (host, once)
                rank = sensitivity_ranking(self.gview, {n: self.w[n] for n in self.sel}, self.sel_layers)
                self.sensitivity = rank
                self.update_layers = sorted(l for l, _ in rank[: t.sensitivity_topk])
                self._build_update_runs()
            for off, n, offs_dev, ptrs_dev, nseg in self._update_runs:
                self._chk(L.mace_adamw_masked2(self.ctx.h, self.master.data_ptr() + 4 * off,
                                               self.m.data_ptr() + 4 * off, self.v.data_ptr() + 4 * off,
                                               self.grad.data_ptr() + 4 * off, n, offs_dev.data_ptr(),
                                               ptrs_dev.data_ptr(), nseg, t.lr, t.beta1, t.beta2, t.eps,
                                               t.weight_decay, self.adam_step, int(self.adam_vec4), s), "adamw")
            return
        self._chk(L.mace_adamw_masked2(self.ctx.h, self.master.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                                       self.grad.data_ptr(), self.n_sel, self.seg_offsets.data_ptr(),
                                       self.seg_ptrs.data_ptr(), len(self.sel), t.lr, t.beta1, t.beta2, t.eps,
                                       t.weight_decay, self.adam_step, int(self.adam_vec4), s), "adamw")

    def _apply_lora_update(self, local_ft: bool) -> None:
        """Per-tenant AdamW of the adapters: each tenant with fine-tune rows this round (on any replica) takes one
        step with its own step count over its own adapter rows only (mace_adamw_segments); the other tenants'
        adapters and optimizer state stay untouched. Replicas all-reduce the gradient and the set of stepping
        tenants, so every replica applies the same updates."""
        L, s, t = self.ctx.L, self._s, self.tcfg
        present = np.zeros(self.n_tenants, np.int32)
        if local_ft:
            present[self._tick_tenants] = 1
        if self.pg is not None:
            if self.grad_allreduce == "bf16":
                g16 = self._g16
                self._chk(L.mace_f32_to_bf16(self.ctx.h, self.grad.data_ptr(), self.n_sel, g16.data_ptr(), s),
                          "grad to bf16")
                torch.distributed.all_reduce(g16, group=self.pg)
                self._chk(L.mace_bf16_to_f32(self.ctx.h, g16.data_ptr(), self.n_sel, self.grad.data_ptr(), s),
                          "grad to f32")
            else:
                torch.distributed.all_reduce(self.grad, group=self.pg)
            mask = torch.from_numpy(present).to(self.dev)
            torch.distributed.all_reduce(mask, op=torch.distributed.ReduceOp.MAX, group=self.pg)
            present = mask.cpu().numpy()
        self.adam_step += 1
        self.last_tenants = [int(u) for u in np.nonzero(present)[0]]
        r, D, R = t.lora_rank, self.cfg.d_model, self.lora_R
        for u in self.last_tenants:
            self.tenant_steps[u] += 1
            vstart, flat, wp, n = self._tenant_seg[u]
            self._chk(L.mace_adamw_segments(self.ctx.h, self.master.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                                            self.grad.data_ptr(), len(self.sel), vstart.data_ptr(), flat.data_ptr(),
                                            wp.data_ptr(), n, t.lr, t.beta1, t.beta2, t.eps, t.weight_decay,
                                            int(self.tenant_steps[u]), int(self.adam_vec4), s), "adamw (tenant)")
            for l in self.sel_layers:  # B of qkv / up: the updated rows back into the augmented weights
                for proj in ("qkv", "up"):
                    bt = self.lw[f"lora.{l}.bt_{proj}"]
                    aug = self.w[f"layers.{l}.{proj}.w"]
                    self._chk(L.mace_lora_bt_scatter(self.ctx.h, bt.data_ptr() + 2 * u * r * bt.shape[1], r,
                                                     bt.shape[1], aug.data_ptr(), D + R, D + u * r, s), "lora scatter")
