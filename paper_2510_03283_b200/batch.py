"""Host-side row tables of one hybrid tick (the ragged batch handed to the device).

Row layout (engine.py:578-584 order): [prefill rows | decode rows | fine-tune rows]
  prefill  uncached prompt suffix of each prefill request, trie-DFS order (cache.dfs_order)
  decode   one row per decode request, id order
  finetune per FT request (id order): [prompt | chosen] then [prompt | rejected]

All integer tables are packed into ONE pinned int32 buffer and moved with one H2D copy per tick.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PAGE = 16

KIND_PREFILL, KIND_DECODE, KIND_FT = 0, 1, 2


@dataclass
class FtPair:
    rid: int
    prompt: list[int]
    chosen: list[int]
    rejected: list[int]
    ref_lp: tuple[float, float] | None = None   # cached pi_ref log-probs (None: computed this tick)
    tenant: int = 0                              # Request.tenant (workload.py:71): whose adapter it trains (LoRA)


@dataclass
class TickBatch:
    tokens: np.ndarray          # [T] int32 (>= 0 literal token, < 0: -(slot+1) -> device last_token[slot])
    pos: np.ndarray             # [T] int32 absolute position (RoPE / learned positions)
    row_seq: np.ndarray         # [T] int32 sequence index
    row_kvi: np.ndarray         # [T] int32 prompt index (prefill) / decode slot index (decode) / -1 (FT)
    seqs: np.ndarray            # [S, 8] int32 MaceSeq
    tc_items: np.ndarray        # [n, 4] int32 (seq, q_head, q_block, 0)
    dec_items: np.ndarray       # [n, 4] int32 (seq, kv_head, chunk, n_chunks)
    dec_slots: np.ndarray       # [n_dec] int32 KV slot of each decode row (alloc + token scatter)
    dec_rows: np.ndarray        # [n_dec] int32 batch row of each decode row
    ptab_slots: np.ndarray      # [u] int32 slots whose prompt page table is (re)written this tick
    ptab_rows: np.ndarray       # [u, maxpp] int32
    page_copies: np.ndarray     # [c, 4] int32 copy-on-diverge (src_group, dst_group, n_tokens, 0)
    ft0: int                    # first FT row
    ft_pairs: list[FtPair] = field(default_factory=list)
    ft_logit_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))  # [R] rows predicting responses
    ft_targets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    pair_rows: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.int32))
    row_ps: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    # FT sub-batch tables (rows relative to ft0) for the pi_ref pass and the backward
    ft_seqs: np.ndarray = field(default_factory=lambda: np.zeros((0, 8), np.int32))
    ft_tc_items: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.int32))
    ft_row_seq: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    bwd_items: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.int32))  # (ft seq, kv_head, kblock, 0)
    row_tenant: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))  # [T] Request.tenant per row
    # accounting (tokens processed by the hybrid iteration)
    n_prefill_tokens: int = 0
    n_decode_tokens: int = 0
    n_ft_tokens: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def T(self) -> int:
        return int(self.tokens.shape[0])

    @property
    def n_dec(self) -> int:
        return int(self.dec_slots.shape[0])

    @property
    def n_ft_rows(self) -> int:
        return self.T - self.ft0

    @property
    def total_tokens(self) -> int:
        return self.n_prefill_tokens + self.n_decode_tokens + self.n_ft_tokens

    def packed(self) -> tuple[np.ndarray, dict[str, tuple[int, tuple[int, ...]]]]:
        """Concatenate every int32 table (16-byte aligned segments) -> (buffer, {name: (offset, shape)})."""
        local_rows = (self.ft_logit_rows - self.ft0).astype(np.int32)
        if self.ft_pairs and all(p.ref_lp is not None for p in self.ft_pairs):
            ref_cached = np.array([p.ref_lp for p in self.ft_pairs], np.float32).view(np.int32)
        else:
            ref_cached = np.zeros((0, 2), np.int32)
        parts = [
            ("tokens", self.tokens), ("pos", self.pos), ("row_seq", self.row_seq), ("row_kvi", self.row_kvi),
            ("seqs", self.seqs), ("tc_items", self.tc_items), ("dec_items", self.dec_items),
            ("dec_slots", self.dec_slots), ("dec_rows", self.dec_rows), ("ptab_slots", self.ptab_slots),
            ("ptab_rows", self.ptab_rows), ("page_copies", self.page_copies),
            ("ft_logit_rows", self.ft_logit_rows), ("ft_targets", self.ft_targets), ("pair_rows", self.pair_rows),
            ("row_ps", self.row_ps), ("ft_seqs", self.ft_seqs), ("ft_tc_items", self.ft_tc_items),
            ("ft_row_seq", self.ft_row_seq), ("bwd_items", self.bwd_items),
            ("ft_local_rows", local_rows), ("ref_cached", ref_cached),  # fp32 bits of cached pi_ref log-probs
            ("row_tenant", self.row_tenant),
        ]
        layout = {}
        off = 0
        for name, a in parts:
            layout[name] = (off, tuple(a.shape))
            off += (a.size + 3) // 4 * 4
        buf = np.zeros(off, np.int32)
        for name, a in parts:
            o, _ = layout[name]
            buf[o: o + a.size] = a.reshape(-1)
        return buf, layout
