"""GpuEngine: the drop-in for the reference's hybrid iteration.

The reference exposes no plugin registry; its override point is ``Engine._execute(plan)``
(/root/reference/pkg/src/macesim/engine.py:573-676), called once per tick with the packed bin of
Alg. 1 (scheduler.py:133-188). ``GpuEngine`` subclasses the UNMODIFIED reference Engine:

  1. it snapshots the bin's pre-tick state and builds ONE ragged batch in the reference's row order
     (prefills in trie-DFS order, decodes by id, fine-tunes by id; engine.py:578-584);
  2. it launches the hybrid step on the B200 (HybridModel.step, all math in libmace_b200.so);
  3. it calls ``super()._execute(plan)`` so every bookkeeping effect (TTFT/TBT, KV MB, head stats,
     prune, ft_step, check_end, retire/requeue, timeline) is the reference's own code;
  4. it mirrors the reference's post-tick KV decisions onto the device (per-head prune trims,
     retirements -> page release; trie evictions via GpuPrefixTrie).

Env: the reference's synthetic AlignmentEnv (decisions bit-identical to the reference), or mode R:
alignenv.DeviceAlignmentEnv, whose pair_loss / ft_step / check_end answers are the device's DPO losses.

Clock modes:
  "P"  parity: the reference cost model drives the clock -> scheduler decisions are bit-identical
       to an unmodified reference run; the GPU executes the same bins for real.
  "M"  measured: the tick duration is the measured device time of the hybrid step (the reference's
       own instrument precedent, engine.py:602-604), via CostProfile.bin_latency (cost_model.py:64-69).
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from .batch import KIND_DECODE, KIND_FT, KIND_PREFILL, PAGE, FtPair, TickBatch
from .config import ModelConfig, TrainConfig
from .hostfast import FastPriorityQueue, NormStream, fast_schedule_iteration, make_bulk_pair_losses
from .hoststats import BatchedHeadStats
from .kvmanager import GpuPrefixTrie, GroupPool, plan_prefill_pages
from .model import HybridModel
from .refpath import ensure_macesim

ensure_macesim()
import macesim.engine as _ref_engine  # noqa: E402
from macesim.cache import dfs_order as _ref_dfs_order  # noqa: E402
from macesim.scheduler import schedule_iteration as _ref_schedule_iteration  # noqa: E402
from macesim.cost_model import CostProfile, WorkloadEstimate  # noqa: E402
from macesim.engine import Engine  # noqa: E402
from macesim.workload import WorkloadType  # noqa: E402


_FAST_ALG1 = os.environ.get("MACE_FAST_ALG1", "1") != "0"  # A/B switch for host profiling


def _dfs_order_hook(trie, pending):
    """Installed once as macesim.engine.dfs_order (engine.py:581-584 calls it by module global).

    A GpuPrefixTrie executing a bin carries that bin's prefill order on the instance (``_bin_order``,
    set and cleared by GpuEngine._execute); every other trie -- a plain reference Engine in the same
    process, another engine between ticks -- gets the reference's whole-trie walk (cache.py:253-273).
    The state lives on the trie instance, so concurrent engines (sweep threads) never see each other's."""
    order = getattr(trie, "_bin_order", None)
    if order is not None:
        return list(order)
    return _ref_dfs_order(trie, pending)


def _schedule_iteration_hook(queue, *args, **kw):
    """Installed once as macesim.engine.schedule_iteration (engine.py:397-402 calls it by module global).

    A FastPriorityQueue owned by a GpuEngine carries its planner on the instance (``_planner``); any other
    queue runs the reference Alg. 1 (scheduler.py:133-188) unchanged."""
    planner = getattr(queue, "_planner", None)
    if planner is not None:
        return planner(queue, *args, **kw)
    return _ref_schedule_iteration(queue, *args, **kw)


if _ref_engine.dfs_order is _ref_dfs_order:  # idempotent on re-import
    _ref_engine.dfs_order = _dfs_order_hook
if _ref_engine.schedule_iteration is _ref_schedule_iteration:
    _ref_engine.schedule_iteration = _schedule_iteration_hook
DECODE_CHUNK_PAGES = 128  # decode contexts longer than 2048 tokens are split into chunks (merged on device)


def synthetic_pair_tokens(seed: int, rid: int, n_c: int, n_r: int, vocab: int) -> tuple[list[int], list[int]]:
    """Builder-defined chosen/rejected content (mace-trace-v1 carries lengths only, workload.py:205,265)."""
    c = np.random.default_rng([seed, 307, rid]).integers(0, vocab, n_c).tolist()
    r = np.random.default_rng([seed, 308, rid]).integers(0, vocab, n_r).tolist()
    return c, r


class _MeasuredProfile(CostProfile):
    """CostProfile whose bin latency is the measured device time of the current tick (mode M).

    CostProfile.bin_latency (cost_model.py:64-69) is the single point where the reference forms a
    tick's duration (engine.py:605-611), so replacing it is the whole measured-clock hook."""

    def bin_latency(self, max_member_lat: float, n_members: int) -> float:
        return self._clock[0]


def measured_profile(profile: CostProfile) -> _MeasuredProfile:
    fields = {k: getattr(profile, k) for k in profile.__dataclass_fields__}
    fields["iter_overhead"] = 0.0
    p = _MeasuredProfile(**fields)
    object.__setattr__(p, "_clock", [0.0])
    return p


def path_dfs_order(pending) -> list:
    """Same order as macesim.cache.dfs_order (cache.py:253-273) without walking the whole trie: a pre-order
    DFS visiting children by ascending first token lists a request when its leaf is reached, i.e. in
    lexicographic order of the first tokens along its root path (a path before its extensions), ties by id."""
    def key(item):
        req, leaf = item
        return ([n.label[0] for n in leaf.path_nodes()], req.id)

    return [r for r, _ in sorted(pending, key=key)]


class TickBudgetReached(Exception):
    """Raised at the END of a tick (after all its effects) to pause Engine.run(); calling run() again
    resumes exactly where it stopped (the loop keeps all state on self, engine.py:680-732)."""


class GpuEngine(Engine):
    def __init__(self, trace, profile, sched_cfg, priority_params, cache_cfg, env, engine_cfg, metrics_horizon=None,
                 *, model: HybridModel, mode: str = "P", seed: int | None = None, record: bool = False,
                 lockstep=None, fast_host: bool = True, norms: str = "synthetic", page_budget: bool | None = None):
        if mode not in ("P", "M"):
            raise ValueError("mode must be 'P' (parity clock) or 'M' (measured clock)")
        if norms not in ("synthetic", "device"):
            raise ValueError("norms must be 'synthetic' (the reference's draws, engine.py:433-442) or 'device'")
        if mode == "M":
            profile = measured_profile(profile)
            engine_cfg = replace(engine_cfg, scheduler_overhead_ms=0.0)
        super().__init__(trace, profile, sched_cfg, priority_params, cache_cfg, env, engine_cfg, metrics_horizon)
        if model.cfg.n_kv_heads != cache_cfg.num_heads:
            raise ValueError("CacheConfig.num_heads must equal the model's KV heads (per-head KV windows)")
        if fast_host and self.queue is not None:  # vectorised re-keying, identical pop order (hostfast.py)
            self.queue = FastPriorityQueue(priority_params, loss_fn=self._loss_of)
            if type(self)._loss_of is Engine._loss_of:  # the reference's loss chain, restated in bulk
                self.queue.bulk_loss = make_bulk_pair_losses(self.env)
            if _FAST_ALG1:  # Alg. 1's restatement, reached through the installed hook (instance state only)
                self.queue._planner = self._fast_plan
        self.model = model
        self.norm_stream = NormStream(self, model.max_slots)
        self.mcfg: ModelConfig = model.cfg
        self.mode = mode
        self.seed = engine_cfg.seed if seed is None else seed
        self.pool = GroupPool(model.prompt_groups)
        if self.trie is not None:
            self.trie = GpuPrefixTrie(profile.decode_kv_mem_per_token, self.pool)
        self.free_slots = list(range(model.max_slots - 1, -1, -1))
        self.slot_of: dict[int, int] = {}
        self.table_of: dict[int, list[int]] = {}
        self.ref_lp: dict[int, tuple[float, float]] = {}
        self._pending_ref: list = []
        self.record = record
        if record:  # the oracle replay compares the decode logits
            model.keep_dec_logits = True
        self.records: list[dict] = []
        self.tick_tokens: list[int] = []
        self.tick_device_ms: list = []      # (start, end) CUDA events per tick (mode M / time_ticks)
        self.tick_decode_ids: list = []     # decode request ids per timed tick (measured TPOT)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self._planned_shared: dict[int, int] = {}
        self._dec_out: list = []
        self.lockstep = lockstep
        self.ticks_done = 0
        self.idle_rounds = 0  # lockstep rounds this replica joined with a drained trace
        self._budget_end: int | None = None
        self.keep_outputs = True
        self.time_ticks = False
        # batched bit-exact head-stats/prune bookkeeping (engine.py:482-532 restated over all rows)
        self.fast_host = fast_host
        cc = cache_cfg
        self.hstats = BatchedHeadStats(model.max_slots, cc.num_heads, cc.norm_window, cc.c_total, cc.prune_window,
                                       cc.norm_tau)
        self._dec_list: list = []
        self._dec_pending: dict | None = None
        self._dec_est = None
        self._pre_est: dict[int, tuple] = {}  # request id -> (cached prefix length, its prefill estimate)
        self._pair_tokens: dict[int, tuple] = {}  # FT request id -> ((id, n_c, n_r), (chosen, rejected))
        self._route_later: list | None = None     # route-backs of the executing bin (pushed after it)
        self._release_later: list | None = None   # KV slots retired by the executing bin (released after it)
        self._tok_arena: torch.Tensor | None = None  # pinned arena for the per-tick greedy-token copies
        self._tok_off = 0
        # head norms feeding HeadStats (engine.py:433-442, cache.py:276-315): the reference's synthetic draws, or the
        # device's real per-head attention-output norms of the tick's last layer (query heads of a KV group
        # combined as sqrt(mean ||o_h||^2)), read back after the tick
        self.norm_source = norms
        self._dev_norms: dict[int, np.ndarray] = {}
        # budget from the page allocator (mode M default): min(the reference's MB budget, the MB the free device
        # pages hold, minus one partial page per live request and head) -- the real pools can never be overrun
        self.page_budget = (mode == "M") if page_budget is None else page_budget

    # ------------------------------------------------------------------ helpers
    def _slot(self, rid: int) -> int:
        if rid not in self.slot_of:
            if not self.free_slots:
                raise RuntimeError("out of KV slots (raise HybridModel max_slots)")
            self.slot_of[rid] = self.free_slots.pop()
        return self.slot_of[rid]

    def _token_slots(self, n: int) -> torch.Tensor:
        """n int32 slots of pinned host memory for this tick's greedy tokens: carved from a pinned arena (the
        tokens are kept for decoded_tokens() anyway), a new arena when the current one is full."""
        a = self._tok_arena
        if a is None or self._tok_off + n > a.numel():
            a = self._tok_arena = torch.empty(max(1 << 16, n), dtype=torch.int32, pin_memory=True)
            self._tok_off = 0
        t = a[self._tok_off: self._tok_off + n]
        self._tok_off += n
        return t

    def _resolve_ref(self) -> None:
        for host, ev, rids in self._pending_ref:
            ev.synchronize()
            arr = host.numpy()
            for i, rid in enumerate(rids):
                self.ref_lp[rid] = (float(arr[i, 0]), float(arr[i, 1]))
        self._pending_ref.clear()

    # ------------------------------------------------------------------ batch building
    def build_batch(self, prefills, decodes, fts) -> TickBatch:
        """Row tables of one tick (numpy-vectorised; the per-row Python is the reference's, not ours)."""
        c = self.mcfg
        Hq, Hkv = c.n_heads, c.n_kv_heads
        i32 = np.int32
        tok_seg, pos_seg, seq_seg, kvi_seg, ten_seg = [], [], [], [], []
        seqs: list[tuple] = []  # sequence rows not yet in seq_blocks
        seq_blocks: list[np.ndarray] = []
        n_seq = 0  # sequences before `seqs`
        tc_seg = []
        ptab_slots, ptab_rows, copies = [], [], []
        n_rows = 0
        n_pre = n_ft = 0
        pending_cached: set[int] = set()
        fresh: set[int] = set()
        self._planned_shared = {}
        hq_grid = np.arange(Hq, dtype=i32)

        blk = 256 if getattr(self.model, "attn_pairs", False) else 128  # query rows per tensor-core attention item

        def tc_block(si, q_len, kv_len):
            """(seq, q head, q block, KV tiles the block visits): one item of the tensor-core attention each; a
            block is 128 query rows, or a PAIR of them (256 rows, csrc/attention_fa2.cu) when model.attn_pairs."""
            nb = (q_len + blk - 1) // blk
            g = np.empty((Hq * nb, 4), i32)
            g[:, 0] = si
            g[:, 1] = np.repeat(hq_grid, nb)
            qb = np.tile(np.arange(nb, dtype=i32), Hq)
            g[:, 2] = qb
            g[:, 3] = (kv_len - q_len + np.minimum(qb * blk + blk - 1, q_len - 1)) // 128 + 1
            return g

        def lpt(items):
            """longest-first launch order (causal blocks differ in KV tiles): the grid tail is short blocks"""
            return items[np.argsort(-items[:, 3], kind="stable")] if items.shape[0] > 1 else items

        # ---- prefill rows (trie-DFS order): uncached suffix of each prompt
        for req in prefills:
            rs = self.state[req.id]
            slot = self._slot(req.id)
            P = len(req.prompt_tokens)
            shared, start, table, cps = plan_prefill_pages(self.trie, self.pool, rs.leaf, P, pending_cached, fresh)
            self._planned_shared[req.id] = shared
            self.table_of[req.id] = table
            ptab_slots.append(slot)
            ptab_rows.append(table)
            copies += [(s_, d_, n_, 0) for s_, d_, n_ in cps]
            q = P - start
            if q <= 0:
                continue
            si = n_seq + len(seqs)
            seqs.append((KIND_PREFILL, n_rows, q, slot, P, P, -1, 0))
            tc_seg.append(tc_block(si, q, P))
            tok_seg.append(np.asarray(req.prompt_tokens[start:], i32))
            ten_seg.append(np.full(q, req.tenant, i32))
            r = np.arange(start, P, dtype=i32)
            pos_seg.append(r)
            kvi_seg.append(r)
            seq_seg.append(np.full(q, si, i32))
            n_rows += q
            n_pre += P - shared  # tokens the reference charges (engine.py:449-450)
        # ---- decode rows (id order): one row each
        n_dec = len(decodes)
        dec_items = np.zeros((0, 4), i32)
        dec_slots = np.zeros(0, i32)
        dec_rows = np.zeros(0, i32)
        if n_dec:
            slot_of = self.slot_of
            info = np.array([(len(pt), r.decode_pos, slot_of[r.id], pt[-1])
                             for r in decodes for pt in (r.prompt_tokens,)], i32).reshape(n_dec, 4)
            P, k0, dec_slots, last = info[:, 0], info[:, 1], info[:, 2], info[:, 3]
            si0 = n_seq + len(seqs)
            dec_rows = np.arange(n_rows, n_rows + n_dec, dtype=i32)
            sarr = np.zeros((n_dec, 8), i32)
            sarr[:, 0] = KIND_DECODE
            sarr[:, 1] = dec_rows
            sarr[:, 2] = 1
            sarr[:, 3] = dec_slots
            sarr[:, 4] = P - 1
            sarr[:, 6] = np.arange(n_dec, dtype=i32)
            seq_blocks.append(np.asarray(seqs, i32).reshape(-1, 8))  # rows so far, then the decode block
            seq_blocks.append(sarr)
            seqs = []
            n_seq = si0 + n_dec
            tok_seg.append(np.where(k0 == 0, last, -(dec_slots + 1)).astype(i32))
            ten_seg.append(np.fromiter((r.tenant for r in decodes), i32, n_dec))
            dpos = (P - 1 + k0).astype(i32)
            if c.family == "gpt2" and int(dpos.max()) >= c.max_pos:
                raise ValueError(f"decode position {int(dpos.max())} >= {c.name}'s {c.max_pos} learned positions "
                                 "(cap prompt length + max_decode_steps)")
            pos_seg.append(dpos)
            seq_seg.append(np.arange(si0, si0 + n_dec, dtype=i32))
            kvi_seg.append(k0)
            n_rows += n_dec
            # decode attention work items: (seq, kv head, chunk << 16 | n_chunks, partial base), LPT order
            npp = (P - 1 + PAGE - 1) // PAGE
            nch = np.maximum(1, -(-npp // DECODE_CHUNK_PAGES))
        if n_dec and int(nch.max()) == 1:
            # every context fits one chunk: one item per (decode, kv head); a stable sort of the decodes by
            # pages, heads ascending within each, is the stable sort of the expanded items
            o = np.argsort(-(npp + k0 // PAGE + 1), kind="stable").astype(i32)
            dec_items = np.empty((n_dec * Hkv, 4), i32)
            dec_items[:, 0] = np.repeat(si0 + o, Hkv)
            dec_items[:, 1] = np.tile(np.arange(Hkv, dtype=i32), n_dec)
            dec_items[:, 2] = 1
            dec_items[:, 3] = 0
        elif n_dec:
            per = -(-npp // nch)
            n_it = nch * Hkv
            seq_i = np.repeat(np.arange(si0, si0 + n_dec, dtype=i32), n_it)
            total_it = int(n_it.sum())
            within = (np.arange(total_it, dtype=i32) - np.repeat(np.cumsum(n_it) - n_it, n_it)).astype(i32)
            nch_r = np.repeat(nch, n_it)
            per_r = np.repeat(per, n_it)
            npp_r = np.repeat(npp, n_it)
            head = within // nch_r
            ch = within % nch_r
            multi = nch_r > 1
            # partial slots: consecutive per (decode, head) for multi-chunk items
            starts = np.cumsum(np.where(nch > 1, n_it, 0)) - np.where(nch > 1, n_it, 0)
            base = np.repeat(starts, n_it) + head * nch_r
            base = np.where(multi, base, 0)
            pages = np.minimum(per_r, npp_r - ch * per_r) + np.where(ch == nch_r - 1, np.repeat(k0, n_it) // PAGE + 1, 0)
            dec_items = np.stack([seq_i, head, (ch << 16) | nch_r, base], 1).astype(i32)
            dec_items = dec_items[np.argsort(-pages, kind="stable")]
        ft0 = n_rows
        n_tc_inference = int(sum(t.shape[0] for t in tc_seg))
        # ---- fine-tune rows (id order): [prompt | chosen], [prompt | rejected]
        pairs: list[FtPair] = []
        lr_seg, tg_seg, ps_seg, pair_rows = [], [], [], []
        ft_seqs, ft_tc_seg, ft_seq_seg, bwd_seg = [], [], [], []
        n_logit = 0
        if fts:
            self._resolve_ref()
        for p_i, req in enumerate(fts):
            P = len(req.prompt_tokens)
            room = max(1, c.max_pos - P)
            n_c = min(req.pair.tokens_chosen, room)
            n_r = min(req.pair.tokens_rejected, room)
            key = (req.id, n_c, n_r)
            hit = self._pair_tokens.get(req.id)
            if hit is None or hit[0] != key:
                content = getattr(req.pair, "chosen", None)
                if content:  # trace v2 (tracev2.ContentPair): the pair's own responses
                    toks = (list(req.pair.chosen[:n_c]), list(req.pair.rejected[:n_r]))
                else:        # mace-trace-v1 carries lengths only: builder-defined synthetic content
                    toks = synthetic_pair_tokens(self.seed, req.id, n_c, n_r, c.vocab)
                hit = self._pair_tokens[req.id] = (key, toks)
            chs, rjs = hit[1]
            pairs.append(FtPair(req.id, req.prompt_tokens, chs, rjs, self.ref_lp.get(req.id), req.tenant))
            # ONE sequence per pair, [prompt | chosen | prompt[-1] | rejected]: the prompt rows are computed once for
            # both responses. The rejected branch re-enters at position P-1 with its own copy of the last prompt
            # token and, through the sequence's key hole [P-1, P + n_c), sees prompt[:-1], that copy and itself --
            # exactly the keys of a separate [prompt | rejected] sequence (MaceSeq hole0 / hole_len).
            n_c, n_r = len(chs), len(rjs)
            n = P + n_c + 1 + n_r
            h0, hl = P - 1, 1 + n_c
            si = n_seq + len(seqs)
            q0 = n_rows
            seqs.append((KIND_FT, q0, n, -1, 0, n, h0, hl))
            tc_seg.append(tc_block(si, n, n))
            fs = len(ft_seqs)
            ft_seqs.append((KIND_FT, q0 - ft0, n, -1, 0, n, h0, hl))
            ft_tc_seg.append(tc_block(fs, n, n))
            kblk = 128 if c.head_dim >= 64 else 64  # key block of the backward kernel (csrc/backward.cu)
            nkb = (n + kblk - 1) // kblk
            bw = np.zeros((Hkv * nkb, 4), i32)
            bw[:, 0] = fs
            bw[:, 1] = np.repeat(np.arange(Hkv, dtype=i32), nkb)
            bw[:, 2] = np.tile(np.arange(nkb, dtype=i32), Hkv)
            bw[:, 3] = nkb - bw[:, 2]  # query blocks the key block walks (LPT key)
            bwd_seg.append(bw)
            prompt = list(req.prompt_tokens)
            tok_seg.append(np.asarray(prompt + list(chs) + prompt[-1:] + list(rjs), i32))
            pos_seg.append(np.concatenate([np.arange(P + n_c, dtype=i32), np.arange(P - 1, P + n_r, dtype=i32)]))
            seq_seg.append(np.full(n, si, i32))
            kvi_seg.append(np.full(n, -1, i32))
            ten_seg.append(np.full(n, req.tenant, i32))
            ft_seq_seg.append(np.full(n, fs, i32))
            # logit rows: chosen[i] is predicted at row P-1+i, rejected[i] at row P+n_c+i (the copy of prompt[-1] first)
            pr = [n_logit, n_c, n_logit + n_c, n_r]
            lr_seg.append(np.arange(q0 + P - 1, q0 + P - 1 + n_c, dtype=i32))
            lr_seg.append(np.arange(q0 + P + n_c, q0 + P + n_c + n_r, dtype=i32))
            tg_seg.append(np.asarray(chs, i32))
            tg_seg.append(np.asarray(rjs, i32))
            ps_seg.append(np.full(n_c, 2 * p_i, i32))
            ps_seg.append(np.full(n_r, 2 * p_i + 1, i32))
            n_logit += n_c + n_r
            n_rows += n
            n_ft += n
            pair_rows.append(pr)

        def cat(segs, tail=None):
            if not segs:
                return np.zeros((0,) + ((tail,) if tail else ()), i32)
            return np.concatenate(segs).astype(i32, copy=False)

        tokens = cat(tok_seg)
        if tokens.size and int(tokens.max()) >= c.vocab:
            raise ValueError(f"token id {int(tokens.max())} >= model vocab {c.vocab} "
                             "(TraceConfig.vocab_size must not exceed the model's vocabulary)")

        def arr(x, tail):
            a = np.asarray(x, dtype=i32)
            return a.reshape(-1, tail)

        maxpp = self.model.maxpp
        pt = np.zeros((len(ptab_rows), maxpp), i32)
        for i, t in enumerate(ptab_rows):
            if len(t) > maxpp:
                raise RuntimeError("prompt longer than max_prompt_len")
            pt[i, : len(t)] = t
        tc_all = cat(tc_seg, 4)
        tc_all = np.concatenate([lpt(tc_all[:n_tc_inference]), lpt(tc_all[n_tc_inference:])])
        return TickBatch(
            tokens=tokens, pos=cat(pos_seg), row_seq=cat(seq_seg), row_kvi=cat(kvi_seg),
            seqs=np.concatenate(seq_blocks + [arr(seqs, 8)]) if seq_blocks else arr(seqs, 8), tc_items=tc_all, dec_items=dec_items,
            dec_slots=dec_slots.astype(i32), dec_rows=dec_rows, ptab_slots=np.asarray(ptab_slots, i32), ptab_rows=pt,
            page_copies=arr(copies, 4), ft0=ft0, ft_pairs=pairs, ft_logit_rows=cat(lr_seg),
            ft_targets=cat(tg_seg), pair_rows=arr(pair_rows, 4), row_ps=cat(ps_seg),
            ft_seqs=arr(ft_seqs, 8), ft_tc_items=lpt(cat(ft_tc_seg, 4)), ft_row_seq=cat(ft_seq_seg),
            bwd_items=lpt(cat(bwd_seg, 4)), row_tenant=cat(ten_seg), n_prefill_tokens=n_pre, n_decode_tokens=n_dec, n_ft_tokens=n_ft,
            meta={"n_tc_inference": n_tc_inference},
        )

    # ------------------------------------------------------------------ the override point
    def _execute(self, plan) -> None:  # engine.py:573
        bin_ = plan.bin
        prefills = [r for r in bin_.tasks if r.workload is WorkloadType.PREFILL]
        decodes = sorted((r for r in bin_.tasks if r.workload is WorkloadType.DECODE), key=lambda r: r.id)
        fts = sorted((r for r in bin_.tasks if r.workload is WorkloadType.FINETUNE), key=lambda r: r.id)
        if self.trie is not None and len(prefills) > 1:  # identical ordering rule to engine.py:581-584
            pending = [(r, self.state[r.id].leaf) for r in prefills]
            if all(leaf is not None for _, leaf in pending):
                prefills = path_dfs_order(pending)
        batch = self.build_batch(prefills, decodes, fts)
        self._dec_list = decodes
        self._dec_pending = None
        m = self.model
        timed = self.mode == "M" or self.time_ticks
        if timed:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
        ft_global = self.lockstep.any_ft(bool(fts)) if self.lockstep is not None else None
        out = m.step(batch, ft_global=ft_global)
        if timed:
            ev1.record()
        self.h2d_bytes += m.h2d_bytes
        if self.norm_source == "device" and out.head_norm is not None:
            hn = out.head_norm.double().cpu().numpy()  # synchronizes: [n_dec, Hq]
            G = self.mcfg.group
            per_kv = np.sqrt((hn.reshape(hn.shape[0], -1, G) ** 2).mean(-1))
            self._dev_norms = {r.id: per_kv[i] for i, r in enumerate(decodes)}
            self.d2h_bytes += hn.size * 4
        observe = getattr(self.env, "observe", None)  # mode R (alignenv.DeviceAlignmentEnv): the device DPO losses
        if observe is not None and fts and out.ft_loss is not None:
            observe([r.id for r in fts], out.ft_loss, out.ft_margin)
            self.d2h_bytes += 8 * len(fts)
        if self.mode == "M":
            ev1.synchronize()
            self.profile._clock[0] = ev0.elapsed_time(ev1)
        # ---- the reference's own bookkeeping for this bin (timeline, metrics, KV MB, prune, ft_step)
        # the reference orders this bin's prefills with dfs_order, a walk of the WHOLE trie (cache.py:253-273);
        # the order is already known (path_dfs_order, equal by construction and by tests/test_host_cpu.py) and
        # is handed over on this engine's own trie instance (_dfs_order_hook)
        if self.trie is not None:
            self.trie._bin_order = prefills
        defer = isinstance(self.queue, FastPriorityQueue)
        self._route_later = [] if defer else None
        self._release_later = []
        try:
            super()._execute(plan)
        finally:
            if self.trie is not None:
                self.trie._bin_order = None
            later, self._route_later = self._route_later, None
            if later:  # the bin's route-backs, pushed together at the clock they were issued at
                self.queue.push_many(later, self.clock)
            rel, self._release_later = self._release_later, None
            if rel:  # retired rows' KV slots (before any later tick can reuse them)
                m.release_slots(rel)
        # ---- mirror post-tick KV decisions onto the device (retired requests were released already)
        live_dec = [r for r in decodes if r.id in self.slot_of]
        if self.pruning and live_dec:
            slots = np.array([self.slot_of[r.id] for r in live_dec], np.int32)
            kept = np.array([self.state[r.id].kept for r in live_dec], np.int32)
            m.apply_trim(slots, kept)
        if out.dec_tokens is not None and self.keep_outputs:
            host = self._token_slots(batch.n_dec)
            host.copy_(out.dec_tokens, non_blocking=True)
            self.d2h_bytes += batch.n_dec * 4
            self._dec_out.append(([r.id for r in decodes], host))
        if fts and out.ref_lp is not None:
            host = torch.empty(len(fts), 2, dtype=torch.float32, pin_memory=True)
            host.copy_(out.ref_lp, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._pending_ref.append((host, ev, [r.id for r in fts]))
            self.d2h_bytes += len(fts) * 8
        self.tick_tokens.append(batch.total_tokens)
        if timed:
            self.tick_device_ms.append((ev0, ev1))
            self.tick_decode_ids.append([r.id for r in decodes])
        self.last_batch = batch
        if self.record:  # host copies for the oracle replay (tests only; synchronizes)
            torch.cuda.current_stream().synchronize()
            rec = dict(tick=self.tick_index - 1, batch=batch,
                       kept_post={self.slot_of[r.id]: list(self.state[r.id].kept) for r in live_dec if self.pruning},
                       dec_tokens=None if out.dec_tokens is None else out.dec_tokens.cpu().numpy().copy(),
                       dec_logits=None if out.dec_tokens is None else m.dec_logits[: batch.n_dec, : self.mcfg.vocab].cpu().clone())
            if fts:
                rec.update(ft_loss=out.ft_loss.cpu().numpy().copy(), ft_margin=out.ft_margin.cpu().numpy().copy(),
                           ft_lp=out.ft_lp.cpu().numpy().copy(), ref_lp=out.ref_lp.cpu().numpy().copy(),
                           grad={n: t.cpu().clone() for n, t in m.gview.items()},
                           tenants=list(getattr(m, "last_tenants", [])),
                           tenant_steps=m.tenant_steps.copy() if m.lora else None,
                           master=m.master.cpu().clone(), adam_m=m.m.cpu().clone(), adam_v=m.v.cpu().clone())
            self.records.append(rec)
        self._after_tick()

    def _after_tick(self) -> None:
        self.ticks_done += 1
        if self._budget_end is not None and self.ticks_done >= self._budget_end:
            raise TickBudgetReached()

    def run_ticks(self, n: int) -> int:
        """Advance the reference loop by exactly n executed ticks (fewer if the trace drains).

        Lockstep replicas (N > 1): every tick round is one Lockstep.tick agreement. A rank whose trace has
        drained keeps joining the rounds idle -- contributing zero gradients to every fine-tune update the
        others run (HybridModel.idle_update) -- until n rounds have passed or no rank has work left, so no
        rank ever waits on a collective the others will not issue. The selected weights of all replicas are
        then compared by checksum (they must be bit-identical)."""
        start = self.ticks_done
        self._budget_end = start + n
        try:
            self.run()
        except TickBudgetReached:
            pass
        finally:
            self._budget_end = None
        done = self.ticks_done - start
        lock = self.lockstep
        if lock is not None and getattr(lock, "active", False):
            rounds = done
            while rounds < n:
                any_ft, any_active = lock.tick(False, active=False)
                if not any_active:
                    break
                if any_ft:
                    self.model.idle_update()
                rounds += 1
            self.idle_rounds += rounds - done
            lock.assert_equal(self.model.weight_checksum(), "selected-parameter weights")
        return done

    def _route_back(self, req, continued_ft):  # engine.py:561 — inside _execute: collected, pushed in bulk
        later = self._route_later
        if later is None:
            return super()._route_back(req, continued_ft)
        later.append(req)

    def _exec_prefill(self, req):  # engine.py:444 — check our plan against the reference's charge
        if self.trie is not None and self.state[req.id].leaf is not None:
            shared = self.trie.cached_prefix_len(req.prompt_tokens)
            planned = self._planned_shared.get(req.id)
            if planned is not None and planned != shared:
                raise AssertionError(f"req {req.id}: planned shared prefix {planned} != reference {shared}")
        return super()._exec_prefill(req)

    def _exec_decode(self, req, t_end_ms):  # engine.py:482 — same effects, head stats batched per tick
        pend = self._dec_pending
        if pend is None:
            if not (self.fast_host and self.pruning) or self.state[req.id].head_stats is None:
                return super()._exec_decode(req, t_end_ms)
            pend = self._dec_pending = self._batch_head_stats()
        hit = pend.get(req.id)
        if hit is None:  # no head stats for this row: the reference path (engine.py:530-532)
            return super()._exec_decode(req, t_end_ms)
        kept, released = hit
        rs = self.state[req.id]
        req.decode_pos += 1
        metrics = self.metrics
        metrics.decoded_tokens += 1
        if rs.first_token_ms is None:
            rs.first_token_ms = t_end_ms
            metrics.ttft_ms[req.id] = t_end_ms - req.arrival_time * 1000.0
            metrics.tbt_ms[req.id] = []
        else:
            metrics.tbt_ms[req.id].append(t_end_ms - rs.last_token_ms)
        rs.last_token_ms = t_end_ms
        heads, per_head, grown = self._dec_consts
        rs.kept = kept
        self.slots_created += heads
        rs.resident_kv_mb += grown
        self._resident_kv_total += grown
        if released:
            self.slots_released += released
            freed = released * per_head
            rs.resident_kv_mb -= freed
            self._resident_kv_total -= freed
            self.timeline.append({"kind": "cache_event", "t": self.clock, "event": "prune", "req_id": req.id,
                                  "bytes_mb": -freed, "slots": released})

    def _batch_head_stats(self) -> dict:
        """Head-stats + allocation + prune for every decode row of this tick (id order)."""
        heads = self.cache_cfg.num_heads
        per_head = self.profile.decode_kv_mem_per_token / heads  # engine.py:494-497, same expressions
        self._dec_consts = (heads, per_head, per_head * heads)
        rows = [r for r in self._dec_list if self.state[r.id].head_stats is not None]
        out: dict = {}
        if not rows:
            return out
        slot_of = self.slot_of
        info = np.array([(slot_of[r.id], r.decode_pos) for r in rows], np.int64).reshape(len(rows), 2)
        slots = np.ascontiguousarray(info[:, 0])
        first = info[:, 1] == 0
        if first.any():
            self.hstats.reset(slots[first])
        steps = info[:, 1] + 1
        if self.norm_source == "device":
            norms = np.stack([self._dev_norms[r.id] for r in rows]).astype(np.float64)
        else:
            norms = self.norm_stream.norms_many(rows, slots)
        kept, released = self.hstats.step(slots, steps, norms)
        return dict(zip([r.id for r in rows], zip(kept.tolist(), released.tolist())))

    def _fast_plan(self, queue, *args, **kw):  # engine.py:397 -> Alg. 1's inlined restatement (hostfast.py)
        return fast_schedule_iteration(queue, *args, dec_est=self._dec_est, **kw)

    def _synth_norms(self, req, rs):  # engine.py:433 — same draws, served from the per-request block stream
        if self.norm_source == "device":
            return self._dev_norms[req.id].tolist()
        return self.norm_stream.norms(req, rs).tolist()

    def _budget(self):  # engine.py:268 — the reference's MB budget, capped by the device pools in page terms
        b = super()._budget()
        if self.page_budget and hasattr(self.model, "kv_mirror"):
            b = min(b, self.page_budget_mb())
        return b

    def page_budget_mb(self) -> float:
        """MB of KV the free device pages can still take, in the profile's units (decode_kv_mem_per_token = the
        model's KV bytes per token / 2^20 in every workload): free prompt groups x 16 tokens plus free decode head
        pages x 16 tokens / H, less one partial prompt group and one partial decode page per head for every live
        request (page rounding)."""
        m = self.model
        kv = self.profile.decode_kv_mem_per_token
        H = m.cfg.n_kv_heads
        live = len(self.live)
        groups = max(0, len(self.pool.free) - live)
        dec = max(0, m.kv_mirror.free - live * H)
        return groups * PAGE * kv + dec * PAGE * kv / H

    def _estimate(self, req):  # engine.py:262 -> cost_model.get_workload (cost_model.py:92-106), same arithmetic
        w = req.workload
        if w is WorkloadType.DECODE:  # constants (cost_model.py:101-102)
            est = self._dec_est
            if est is None:
                est = self._dec_est = super()._estimate(req)
            return est
        if w is WorkloadType.PREFILL and self.fast_host and isinstance(self.trie, GpuPrefixTrie):
            # cost_model.py:95-99 with the memoised cached-prefix walk of a queued prompt
            shared = self.trie.cached_prefix_len_memo(req.id, req.prompt_tokens)
            hit = self._pre_est.get(req.id)
            if hit is not None and hit[0] == shared:
                return hit[1]
            effective = max(0, len(req.prompt_tokens) - shared)
            p = self.profile
            est = WorkloadEstimate(mem=(p.prefill_mem_per_token + p.decode_kv_mem_per_token) * effective,
                                   lat=p.prefill_lat_per_token * effective)
            self._pre_est[req.id] = (shared, est)
            return est
        return super()._estimate(req)

    def _retire(self, req, t_end_ms, rejected=False):  # engine.py:538
        self.norm_stream.drop(req.id)
        self._pre_est.pop(req.id, None)
        self._pair_tokens.pop(req.id, None)
        if isinstance(self.trie, GpuPrefixTrie):
            self.trie.forget(req.id)
        super()._retire(req, t_end_ms, rejected)
        slot = self.slot_of.pop(req.id, None)
        table = self.table_of.pop(req.id, None)
        if table is not None:
            for g in table:
                self.pool.decref(g)
        if slot is not None:
            if self._release_later is not None:  # inside the bin's bookkeeping: one release call per tick
                self._release_later.append(slot)
            else:
                self.model.release_slots([slot])
            self.free_slots.append(slot)

    # ------------------------------------------------------------------ results
    def decoded_tokens(self) -> dict[int, list[int]]:
        torch.cuda.current_stream().synchronize()
        out: dict[int, list[int]] = {}
        for ids, host in self._dec_out:
            arr = host.numpy()
            for i, rid in enumerate(ids):
                out.setdefault(rid, []).append(int(arr[i]))
        return out

    def measured_tbt_ms(self, first: int = 0) -> list[float]:
        """Time between consecutive tokens of every request, measured on the device clock: the gap between the
        end events of the two ticks that emitted them (includes any time the device waited on the host). The
        reference's TBT (engine.py:130-143) on the measured clock; ticks from index ``first`` of the timed list."""
        torch.cuda.current_stream().synchronize()
        last: dict[int, int] = {}
        out = []
        for i in range(first, len(self.tick_device_ms)):
            for rid in self.tick_decode_ids[i]:
                j = last.get(rid)
                if j is not None:
                    out.append(self.tick_device_ms[j][1].elapsed_time(self.tick_device_ms[i][1]))
                last[rid] = i
        return out

    def device_ms(self) -> list[float]:
        torch.cuda.current_stream().synchronize()
        return [a.elapsed_time(b) for a, b in self.tick_device_ms]
