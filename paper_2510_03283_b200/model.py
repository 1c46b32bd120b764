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
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from ._lib import Ctx, MaceKvLayout
from .batch import PAGE, TickBatch
from .config import ModelConfig, TrainConfig, selected_param_names


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
    ):
        self.cfg, self.tcfg = cfg, tcfg
        self.ctx = ctx or Ctx(device)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.current_stream(self.dev)
        self.pg = process_group
        d, L = cfg.d_model, cfg.n_layers
        self.w = {n: t.to(self.dev, torch.bfloat16).contiguous() for n, t in weights.items()}
        # ---- selected parameters: flat fp32 master / m / v / grad + segment table for masked AdamW
        self.sel = selected_param_names(cfg, tcfg)
        self.sel_layers = tcfg.selected_layers(cfg)
        self.l_min = min(self.sel_layers)
        sizes = [self.w[n].numel() for n in self.sel]
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.n_sel = int(offs[-1])
        self.master = torch.cat([self.w[n].float().reshape(-1) for n in self.sel])
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.grad = torch.zeros_like(self.master)
        self.gview = {n: self.grad[offs[i]: offs[i + 1]].view(self.w[n].shape) for i, n in enumerate(self.sel)}
        self.seg_offsets = torch.from_numpy(offs).to(self.dev)
        self.seg_ptrs = torch.tensor([self.w[n].data_ptr() for n in self.sel], dtype=torch.int64, device=self.dev)
        self.adam_step = 0
        self.ref_w = {n: self.w[n].clone() for n in self.sel}  # pi_ref frozen at init
        # ---- RoPE tables (fp64 on host -> fp32)
        half = cfg.head_dim // 2
        inv = cfg.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim)
        ang = np.arange(cfg.max_pos, dtype=np.float64)[:, None] * inv[None, :]
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
        self.decode_pages = decode_pages
        self.pages_per_layer = prompt_groups * H + decode_pages
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
        self.free_stack = torch.arange(prompt_groups * H, self.pages_per_layer, **i32)
        self.free_top = torch.tensor([decode_pages], **i32)
        self.last_token = torch.zeros(max_slots, **i32)
        self.dec_counters = torch.zeros(max_slots * H, **i32)  # decode chunk-merge counters (self-cleaning)
        self.dec_work = torch.zeros(1, dtype=torch.int64, device=self.dev)  # decode ticket counter (monotonic)
        self.decode_impl = 0  # 0 auto (tcgen05 swap-AB for GQA, CUDA-core streaming for MHA), 1, 2 forced
        self.kv = MaceKvLayout(
            ptab=self.ptab.data_ptr(), max_prompt_pages=self.maxpp, dtab=self.dtab.data_ptr(),
            max_dec_pages=self.maxdp, dec_base=self.dec_base.data_ptr(), dec_first=self.dec_first.data_ptr(),
            dec_end=self.dec_end.data_ptr(), free_stack=self.free_stack.data_ptr(),
            free_top=self.free_top.data_ptr(), stack_cap=decode_pages, n_kv_heads=H,
        )
        self._cap = 0
        self._ft_cap = 0
        self._R_cap = 0
        self._ndec_cap = 0
        self.ws = torch.empty(16 << 20, dtype=torch.float32, device=self.dev)  # 64 MB split-K / reduction scratch
        self.tape: list | None = None   # when a list: every device-side call is appended (bench replay)
        self.instrument: list | None = None  # when a list: (ev0, ev1, bytes) per decode-attention launch
        self._attn_bytes = 0
        self.idx = torch.empty(1 << 16, dtype=torch.int32, device=self.dev)

    # ------------------------------------------------------------------ buffers
    def _ensure(self, T: int, n_ft: int, R: int, n_dec: int) -> None:
        c, dev = self.cfg, self.dev
        bf, f32 = dict(dtype=torch.bfloat16, device=dev), dict(dtype=torch.float32, device=dev)
        if T > self._cap:
            cap = max(T, int(self._cap * 1.5), 256)
            self.x = torch.empty(cap, c.d_model, **f32)
            self.h = torch.empty(cap, c.d_model, **bf)
            self.qkv = torch.empty(cap, c.qkv_dim, **bf)
            self.o = torch.empty(cap, c.n_heads * c.head_dim, **bf)
            self.lse = torch.empty(cap, c.n_heads, **f32)
            self.hn = torch.empty(cap, c.n_heads, **f32)
            self.u = torch.empty(cap, c.up_dim, **bf)
            self.a = torch.empty(cap, c.ffn, **bf)
            self._cap = cap
        if n_ft > self._ft_cap:
            cap = max(n_ft, int(self._ft_cap * 1.5), 128)
            self.sav = {}
            for l in self.sel_layers:
                self.sav[l] = dict(
                    x_in=torch.empty(cap, c.d_model, **f32), h1=torch.empty(cap, c.d_model, **bf),
                    qkv=torch.empty(cap, c.qkv_dim, **bf), o=torch.empty(cap, c.n_heads * c.head_dim, **bf),
                    lse=torch.empty(cap, c.n_heads, **f32), x_mid=torch.empty(cap, c.d_model, **f32),
                    h2=torch.empty(cap, c.d_model, **bf), u=torch.empty(cap, c.up_dim, **bf),
                    a=torch.empty(cap, c.ffn, **bf),
                )
            # ref-pass + backward scratch (FT rows only)
            self.rx = torch.empty(cap, c.d_model, **f32)
            self.rx2 = torch.empty(cap, c.d_model, **f32)
            self.x_lmin = torch.empty(cap, c.d_model, **f32)
            self.rlse = torch.empty(cap, c.n_heads, **f32)
            self.rh = torch.empty(cap, c.d_model, **bf)
            self.rqkv = torch.empty(cap, c.qkv_dim, **bf)
            self.ro = torch.empty(cap, c.n_heads * c.head_dim, **bf)
            self.ru = torch.empty(cap, c.up_dim, **bf)
            self.ra = torch.empty(cap, c.ffn, **bf)
            self.dx = torch.empty(cap, c.d_model, **f32)
            self.dy16 = torch.empty(cap, c.d_model, **bf)
            self.df = torch.empty(cap, max(c.ffn, c.up_dim, c.qkv_dim, c.n_heads * c.head_dim), **f32)
            self.da16 = torch.empty(cap, c.ffn, **bf)
            self.du16 = torch.empty(cap, c.up_dim, **bf)
            self.do16 = torch.empty(cap, c.n_heads * c.head_dim, **bf)
            self.dqkv = torch.empty(cap, c.qkv_dim, **f32)
            self.dqkv16 = torch.empty(cap, c.qkv_dim, **bf)
            self.Dbuf = torch.empty(cap, c.n_heads, **f32)
            self._ft_cap = cap
        if R > self._R_cap:
            cap = max(R, int(self._R_cap * 1.5), 64)
            self.ft_h = torch.empty(cap, c.d_model, **bf)
            self.ft_logits = torch.empty(cap, c.vocab, **f32)
            self.vpad = (c.vocab + 7) // 8 * 8  # 16-byte aligned rows for the TMA operand of dX = dlogits . E
            self.dlogits = torch.empty(cap, self.vpad, **bf)
            self.dh = torch.empty(cap, c.d_model, **f32)
            self.row_lse = torch.empty(cap, **f32)
            self.row_lp = torch.empty(cap, **f32)
            self._R_cap = cap
        if n_dec > self._ndec_cap:
            cap = max(n_dec, int(self._ndec_cap * 1.5), 64)
            self.dec_h = torch.empty(cap, c.d_model, **bf)
            self.dec_logits = torch.empty(cap, c.vocab, **f32)
            self.dec_tok = torch.empty(cap, dtype=torch.int32, device=dev)
            self.dec_ws = torch.empty(cap * c.n_kv_heads * 4 * (2 * c.group + c.group * c.head_dim), **f32)
            self._ndec_cap = cap

    def replay(self, tape) -> None:
        """Re-issue a recorded sequence of device calls (bench: device-only throughput)."""
        for op in tape:
            if op[0] == "step":
                self.step(op[1], ft_global=op[2])
            elif op[0] == "trim":
                self.apply_trim(op[1], op[2])
            else:
                self.release_slots(op[1])

    def _upload(self, batch: TickBatch) -> dict[str, torch.Tensor]:
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
        views = {}
        for name, (off, shape) in layout.items():
            cnt = int(np.prod(shape)) if len(shape) else 0
            views[name] = self.idx[off: off + cnt].view(*shape) if cnt else None
        return views

    # ------------------------------------------------------------------ primitive wrappers
    def _chk(self, rc, what):
        self.ctx.check(rc, what)

    @property
    def _s(self) -> int:
        return torch.cuda.current_stream(self.dev).cuda_stream

    def _norm(self, x, ldx, rows, n, wname, W, out, ldo):
        c = self.cfg
        ln = c.family == "gpt2"
        b = W.get(wname[:-2] + ".b") if ln else None
        self._chk(self.ctx.L.mace_norm(self.ctx.h, x.data_ptr(), ldx, _p(rows), n, c.d_model, W[wname].data_ptr(),
                                       _p(b), int(ln), c.norm_eps, out.data_ptr(), ldo, None, self._s), "norm")

    def _gemm(self, a, b, out, mode, bias=None, a_mn=False, b_mn=False):
        ops.gemm(self.ctx, a, b, out, mode=mode, bias=bias, a_mn=a_mn, b_mn=b_mn, workspace=self.ws)

    # ------------------------------------------------------------------ one decoder layer (forward)
    def _layer(self, l, W, T, x, h, qkv, o, u, a, seqs, tc_items, dec_items, row_seq, row_pos, row_kvi,
               paged: bool, lse=None, hn=None, save=None, ft0=0):
        c = self.cfg
        p = f"layers.{l}."
        bias = (lambda n: W[p + n + ".b"]) if c.has_bias else (lambda n: None)
        if save is not None:
            save["x_in"][: T - ft0].copy_(x[ft0:T])
        self._norm(x, c.d_model, None, T, p + "attn_norm.w", W, h, c.d_model)
        self._gemm(h[:T], W[p + "qkv.w"], qkv[:T], "bf16", bias("qkv"))
        lay = self.kv
        kp = self.k_pool[l] if paged else None
        vp = self.v_pool[l] if paged else None
        self._chk(self.ctx.L.mace_rope_kv(self.ctx.h, qkv.data_ptr(), T, c.n_heads, c.n_kv_heads, c.head_dim,
                                          row_pos.data_ptr(), row_seq.data_ptr(), _p(row_kvi), seqs.data_ptr(),
                                          self.cos_t.data_ptr(), self.sin_t.data_ptr(), int(c.family == "llama"),
                                          C.byref(lay), _p(kp), _p(vp), self._s), "rope_kv")
        if self.instrument is not None and dec_items is not None:
            if tc_items is not None:
                ops.attn_fwd(self.ctx, qkv[:T], c.n_heads, c.n_kv_heads, c.head_dim, seqs, tc_items, None, lay,
                             kp, vp, o[:T], lse=lse, head_norm=hn)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.attn_fwd(self.ctx, qkv[:T], c.n_heads, c.n_kv_heads, c.head_dim, seqs, None, dec_items, lay,
                         kp, vp, o[:T], lse=lse, head_norm=hn, dec_workspace=self.dec_ws,
                         dec_counters=self.dec_counters, dec_work=self.dec_work,
                         decode_impl=self.decode_impl)
            e1.record()
            self.instrument.append((e0, e1, self._attn_bytes))
        else:
            ops.attn_fwd(self.ctx, qkv[:T], c.n_heads, c.n_kv_heads, c.head_dim, seqs, tc_items, dec_items, lay,
                         kp, vp, o[:T], lse=lse, head_norm=hn, dec_workspace=self.dec_ws,
                         dec_counters=self.dec_counters, dec_work=self.dec_work,
                         decode_impl=self.decode_impl)
        if save is not None:
            n = T - ft0
            save["h1"][:n].copy_(h[ft0:T])
            save["qkv"][:n].copy_(qkv[ft0:T])
            save["o"][:n].copy_(o[ft0:T])
            save["lse"][:n].copy_(lse[ft0:T])
        self._gemm(o[:T], W[p + "o.w"], x[:T], "f32_add", bias("o"))
        if save is not None:
            save["x_mid"][: T - ft0].copy_(x[ft0:T])
        self._norm(x, c.d_model, None, T, p + "mlp_norm.w", W, h, c.d_model)
        if c.family == "gpt2" and save is None:
            # GELU fused into the up-projection epilogue (no pre-activation needed without a backward)
            self._gemm(h[:T], W[p + "up.w"], a[:T], "bf16_gelu", bias("up"))
        else:
            self._gemm(h[:T], W[p + "up.w"], u[:T], "bf16", bias("up"))
            self._chk(self.ctx.L.mace_act(self.ctx.h, u.data_ptr(), T, c.ffn, int(c.family == "llama"),
                                          a.data_ptr(), self._s), "act")
        if save is not None:
            n = T - ft0
            save["h2"][:n].copy_(h[ft0:T])
            save["u"][:n].copy_(u[ft0:T])
            save["a"][:n].copy_(a[ft0:T])
        self._gemm(a[:T], W[p + "down.w"], x[:T], "f32_add", bias("down"))

    # ------------------------------------------------------------------ tick
    @torch.no_grad()
    def step(self, batch: TickBatch, trim: tuple[np.ndarray, np.ndarray] | None = None,
             ft_global: bool | None = None) -> StepOutputs:
        """Run one hybrid tick on the device (asynchronous; outputs are device tensors).

        ``ft_global``: whether ANY replica has fine-tune rows this tick (lockstep multi-GPU); defaults to
        this replica's own rows."""
        if self.tape is not None:
            self.tape.append(("step", batch, ft_global))
        c = self.cfg
        T, ft0 = batch.T, batch.ft0
        n_ft = T - ft0
        R = int(batch.ft_logit_rows.shape[0])
        n_dec = batch.n_dec
        self._ensure(max(T, 1), max(n_ft, 1), max(R, 1), max(n_dec, 1))
        v = self._upload(batch)
        L = self.ctx.L
        s = self._s
        # ---- page-table maintenance (host page manager decisions -> device)
        if v["ptab_slots"] is not None:
            self._chk(L.mace_kv_set_prompt_tables(self.ctx.h, C.byref(self.kv), v["ptab_slots"].data_ptr(),
                                                  v["ptab_rows"].data_ptr(), batch.ptab_slots.shape[0],
                                                  batch.ptab_rows.shape[1], s), "set_tables")
        if v["page_copies"] is not None:
            self._chk(L.mace_kv_page_copy(self.ctx.h, v["page_copies"].data_ptr(), batch.page_copies.shape[0],
                                          c.n_kv_heads, c.head_dim, self.pages_per_layer, c.n_layers,
                                          self.k_pool.data_ptr(), self.v_pool.data_ptr(), s), "page_copy")
        if n_dec:
            self._chk(L.mace_kv_decode_alloc(self.ctx.h, C.byref(self.kv), v["dec_slots"].data_ptr(), n_dec, s),
                      "decode_alloc")
        if self.instrument is not None and n_dec:
            self._attn_bytes = self.decode_attn_bytes(batch)
        out = StepOutputs(None, None, None, None, None, None)
        if T == 0:
            if ft_global:
                self.apply_update(False)
            return out
        # ---- forward through all layers (one ragged batch)
        self._chk(L.mace_embed(self.ctx.h, v["tokens"].data_ptr(), v["pos"].data_ptr(), self.last_token.data_ptr(),
                               self.w["embed"].data_ptr(), _p(self.w.get("pos_embed")), T, c.d_model,
                               self.x.data_ptr(), s), "embed")
        has_ft = n_ft > 0 and len(batch.ft_pairs) > 0
        n_tc_all = 0 if v["tc_items"] is None else v["tc_items"].shape[0]
        n_tc_inf = int(batch.meta.get("n_tc_inference", n_tc_all))
        for l in range(c.n_layers):
            # FT rows ride in the shared ragged batch below the lowest selected layer; from there on they
            # run as their own sub-batch (policy with saved activations + the pi_ref pass) so the two
            # log-prob paths are kernel-for-kernel identical (margin exactly 0 while pi_theta = pi_ref)
            top = has_ft and l >= self.l_min
            T_l = ft0 if top else T
            if has_ft and l == self.l_min:
                self.x_lmin[:n_ft].copy_(self.x[ft0:T])
            if T_l == 0:
                continue
            tci = v["tc_items"][:n_tc_inf] if top else v["tc_items"]
            if tci is not None and tci.shape[0] == 0:
                tci = None
            hn = self.hn if l == c.n_layers - 1 else None
            self._layer(l, self.w, T_l, self.x, self.h, self.qkv, self.o, self.u, self.a, v["seqs"], tci,
                        v["dec_items"], v["row_seq"], v["pos"], v["row_kvi"], paged=True, hn=hn)
        # ---- decode rows: final norm on gathered rows -> lm_head -> greedy token
        if n_dec:
            self._norm(self.x, c.d_model, v["dec_rows"], n_dec, "final_norm.w", self.w, self.dec_h, c.d_model)
            self._gemm(self.dec_h[:n_dec], self.w["embed"], self.dec_logits[:n_dec], "f32")
            self._chk(L.mace_argmax(self.ctx.h, self.dec_logits.data_ptr(), n_dec, c.vocab, c.vocab,
                                    self.dec_tok.data_ptr(), s), "argmax")
            self._chk(L.mace_scatter_tokens(self.ctx.h, self.dec_tok.data_ptr(), v["dec_slots"].data_ptr(), n_dec,
                                            self.last_token.data_ptr(), s), "scatter_tokens")
            out.dec_tokens = self.dec_tok[:n_dec]
        if trim is not None and trim[0].size:
            self.apply_trim(*trim)
        if has_ft:
            self._ft_step(batch, v, out)
        if has_ft or ft_global:
            self.apply_update(has_ft)
        return out

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
        t_s = torch.from_numpy(np.ascontiguousarray(slots, np.int32)).pin_memory().to(self.dev, non_blocking=True)
        t_k = torch.from_numpy(np.ascontiguousarray(kept, np.int32).reshape(-1)).pin_memory().to(self.dev, non_blocking=True)
        self._keep = (t_s, t_k)  # keep alive until the stream consumes them
        self._chk(self.ctx.L.mace_kv_trim(self.ctx.h, C.byref(self.kv), t_s.data_ptr(), t_k.data_ptr(), n, self._s),
                  "kv_trim")

    def release_slots(self, slots: list[int]) -> None:
        if not slots:
            return
        if self.tape is not None:
            self.tape.append(("release", list(slots)))
        t_s = torch.tensor(slots, dtype=torch.int32).pin_memory().to(self.dev, non_blocking=True)
        self._keep_rel = t_s
        self._chk(self.ctx.L.mace_kv_release(self.ctx.h, C.byref(self.kv), t_s.data_ptr(), len(slots), self._s),
                  "kv_release")

    # ------------------------------------------------------------------ fine-tune rows
    def _lm_rows(self, x, rows, R, W, out_h, logits):
        c = self.cfg
        self._norm(x, c.d_model, rows, R, "final_norm.w", W, out_h, c.d_model)
        self._gemm(out_h[:R], self.w["embed"], logits[:R], "f32")

    def _ft_step(self, batch: TickBatch, v, out: StepOutputs) -> None:
        c, L, s = self.cfg, self.ctx.L, self._s
        T, ft0 = batch.T, batch.ft0
        n = T - ft0
        R = int(batch.ft_logit_rows.shape[0])
        P = len(batch.ft_pairs)
        f32 = dict(dtype=torch.float32, device=self.dev)
        lp = torch.empty(P, 2, **f32)
        ref_lp = torch.empty(P, 2, **f32)
        loss = torch.empty(P, **f32)
        margin = torch.empty(P, **f32)
        coef = torch.empty(P, 2, **f32)
        local_rows = v["ft_logit_rows"] - ft0
        ft_pos = v["pos"][ft0:T]

        def sub_pass(W, x, save: bool):
            x[:n].copy_(self.x_lmin[:n])
            for l in self.sel_layers:
                self._layer(l, W, n, x, self.rh, self.rqkv, self.ro, self.ru, self.ra, v["ft_seqs"], v["ft_tc_items"],
                            None, v["ft_row_seq"], ft_pos, None, paged=False, lse=self.rlse if save else None,
                            save=self.sav[l] if save else None, ft0=0)
            self._lm_rows(x, local_rows, R, W, self.ft_h, self.ft_logits)

        # ---- pi_ref log-probs (once per pair): selected layers with the frozen weights from the shared input
        if any(p.ref_lp is None for p in batch.ft_pairs):
            Wref = dict(self.w)
            Wref.update(self.ref_w)
            sub_pass(Wref, self.rx2, save=False)
            self._chk(L.mace_dpo_fused(self.ctx.h, self.ft_logits.data_ptr(), R, c.vocab, c.vocab,
                                       v["ft_targets"].data_ptr(), v["pair_rows"].data_ptr(), P, v["row_ps"].data_ptr(),
                                       None, 0.0, self.row_lse.data_ptr(), self.row_lp.data_ptr(), ref_lp.data_ptr(),
                                       None, None, None, None, 0, s), "dpo_ref")
        else:
            ref_lp.copy_(torch.tensor([p.ref_lp for p in batch.ft_pairs], dtype=torch.float32), non_blocking=True)
        # ---- policy log-probs (saving activations), DPO loss and dlogits
        sub_pass(self.w, self.rx, save=True)
        self._chk(L.mace_dpo_fused(self.ctx.h, self.ft_logits.data_ptr(), R, c.vocab, c.vocab,
                                   v["ft_targets"].data_ptr(), v["pair_rows"].data_ptr(), P, v["row_ps"].data_ptr(),
                                   ref_lp.data_ptr(), self.tcfg.dpo_beta, self.row_lse.data_ptr(),
                                   self.row_lp.data_ptr(), lp.data_ptr(), loss.data_ptr(), margin.data_ptr(),
                                   coef.data_ptr(), self.dlogits.data_ptr(), self.vpad, s), "dpo")
        out.ft_loss, out.ft_margin, out.ft_lp, out.ref_lp = loss, margin, lp, ref_lp
        # ---- backward: lm_head (tied, frozen) -> final norm -> selected layers top-down
        self.grad.zero_()
        self._gemm(self.dlogits[:R, : c.vocab], self.w["embed"], self.dh[:R], "f32", b_mn=True)
        self.dx[:n].zero_()
        self._norm_bwd(self.rx, local_rows, self.dh, R, "final_norm", self.dx, local_rows)
        for l in reversed(self.sel_layers):
            self._layer_bwd(l, n, v, ft_pos)

    def apply_update(self, local_ft: bool) -> None:
        """Gradient exchange (NCCL all-reduce over the request-stream replicas) and the
        masked AdamW. A replica without FT rows this tick contributes zeros and applies the same
        update, so every replica keeps bit-identical weights."""
        L, s = self.ctx.L, self._s
        if not local_ft:
            self.grad.zero_()
        if self.pg is not None:
            torch.distributed.all_reduce(self.grad, group=self.pg)
        self.adam_step += 1
        t = self.tcfg
        self._chk(L.mace_adamw_masked(self.ctx.h, self.master.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                                      self.grad.data_ptr(), self.n_sel, self.seg_offsets.data_ptr(),
                                      self.seg_ptrs.data_ptr(), len(self.sel), t.lr, t.beta1, t.beta2, t.eps,
                                      t.weight_decay, self.adam_step, s), "adamw")

    def _norm_bwd(self, x, xrows, dy, n, name, dx, dxrows):
        c = self.cfg
        ln = c.family == "gpt2"
        self._chk(self.ctx.L.mace_norm_bwd(self.ctx.h, x.data_ptr(), c.d_model, _p(xrows), dy.data_ptr(), c.d_model, n,
                                           c.d_model, self.w[name + ".w"].data_ptr(), int(ln), c.norm_eps,
                                           dx.data_ptr(), c.d_model, _p(dxrows), self.gview[name + ".w"].data_ptr(),
                                           _p(self.gview.get(name + ".b")), self.ws.data_ptr(),
                                           self.ws.numel() * 4, self._s), "norm_bwd")

    def _colsum(self, y16, n, N, name):
        if name not in self.gview:
            return
        self._chk(self.ctx.L.mace_colsum_bf16(self.ctx.h, y16.data_ptr(), n, N, N, self.gview[name].data_ptr(),
                                              self.ws.data_ptr(), self.ws.numel() * 4, self._s), "colsum")

    def _to16(self, x, n_elems, y):
        self._chk(self.ctx.L.mace_f32_to_bf16(self.ctx.h, x.data_ptr(), n_elems, y.data_ptr(), self._s), "to_bf16")

    def _layer_bwd(self, l, n, v, ft_pos):
        """dx (grad wrt this layer's output, FT rows) -> grad wrt its input; dW of the layer's params."""
        c, L = self.cfg, self.ctx.L
        sv = self.sav[l]
        p = f"layers.{l}."
        d, F, up, W, HO = c.d_model, c.ffn, c.up_dim, c.qkv_dim, c.n_heads * c.head_dim
        g = self.gview
        # MLP: down
        self._to16(self.dx, n * d, self.dy16)
        self._gemm(self.dy16[:n], sv["a"][:n], g[p + "down.w"], "f32_add", a_mn=True, b_mn=True)
        self._colsum(self.dy16, n, d, p + "down.b")
        self._gemm(self.dy16[:n], self.w[p + "down.w"], self.da16[:n], "bf16", b_mn=True)
        self._chk(L.mace_act_bwd(self.ctx.h, sv["u"].data_ptr(), self.da16.data_ptr(), n, F,
                                 int(c.family == "llama"), self.du16.data_ptr(), self._s), "act_bwd")
        # MLP: up
        self._gemm(self.du16[:n], sv["h2"][:n], g[p + "up.w"], "f32_add", a_mn=True, b_mn=True)
        self._colsum(self.du16, n, up, p + "up.b")
        dh = self.df[:n, :d]
        self._gemm(self.du16[:n], self.w[p + "up.w"], self.df[:n, :d], "f32", b_mn=True)
        self._norm_bwd_local(sv["x_mid"], self.df, n, p + "mlp_norm")
        # attention: o projection
        self._to16(self.dx, n * d, self.dy16)
        self._gemm(self.dy16[:n], sv["o"][:n], g[p + "o.w"], "f32_add", a_mn=True, b_mn=True)
        self._colsum(self.dy16, n, d, p + "o.b")
        self._gemm(self.dy16[:n], self.w[p + "o.w"], self.do16[:n], "bf16", b_mn=True)
        # attention core
        self.dqkv[:n].zero_()
        self._chk(L.mace_attn_bwd(self.ctx.h, sv["qkv"].data_ptr(), sv["o"].data_ptr(), self.do16.data_ptr(),
                                  sv["lse"].data_ptr(), n, c.n_heads, c.n_kv_heads, c.head_dim,
                                  v["ft_seqs"].data_ptr(), v["bwd_items"].data_ptr(), v["bwd_items"].shape[0], 0,
                                  self.Dbuf.data_ptr(), self.dqkv.data_ptr(), self._s), "attn_bwd")
        if c.family == "llama":
            self._chk(L.mace_rope_bwd(self.ctx.h, self.dqkv.data_ptr(), n, c.n_heads, c.n_kv_heads, c.head_dim,
                                      ft_pos.data_ptr(), self.cos_t.data_ptr(), self.sin_t.data_ptr(), self._s),
                      "rope_bwd")
        self._to16(self.dqkv, n * W, self.dqkv16)
        self._gemm(self.dqkv16[:n], sv["h1"][:n], g[p + "qkv.w"], "f32_add", a_mn=True, b_mn=True)
        self._colsum(self.dqkv16, n, W, p + "qkv.b")
        self._gemm(self.dqkv16[:n], self.w[p + "qkv.w"], self.df[:n, :d], "f32", b_mn=True)
        self._norm_bwd_local(sv["x_in"], self.df, n, p + "attn_norm")

    def _norm_bwd_local(self, x, dyf, n, name):
        """dx += norm_bwd(x, dy) for FT-local rows; dy rows live in dyf[:, :d] (row stride = dyf.shape[1])."""
        c = self.cfg
        ln = c.family == "gpt2"
        self._chk(self.ctx.L.mace_norm_bwd(self.ctx.h, x.data_ptr(), c.d_model, None, dyf.data_ptr(), dyf.shape[1], n,
                                           c.d_model, self.w[name + ".w"].data_ptr(), int(ln), c.norm_eps,
                                           self.dx.data_ptr(), c.d_model, None, self.gview[name + ".w"].data_ptr(),
                                           _p(self.gview.get(name + ".b")), self.ws.data_ptr(),
                                           self.ws.numel() * 4, self._s), "norm_bwd")
