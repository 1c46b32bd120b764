"""Sampled-tick CPU execution of the hybrid iteration (test / bench infrastructure only -- see
oracle/model_ref.py's header: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg and
--impl reference arm use this module; the product never imports it).

Why sampled: one prefill-heavy Llama-3-8B tick of config C4 holds ~20k prefill rows, ~250 decode rows and
~10k fine-tune rows -- hundreds of TFLOP, i.e. minutes of fp32 CPU time per tick. BASELINE.md §2 asks for the
CPU path "on a sampled subset of ticks for C3-C5"; this module is that sample, row-granular:

  * the tick's bin is the UNMODIFIED reference scheduler's (macesim.engine.Engine, mode-P clock), captured by
    ``composition`` from the bin the reference hands to Engine._execute (engine.py:573-584): prefill rows = the
    uncached prompt suffix the reference charges (cache.py:164-184), decode rows = one per decode request,
    fine-tune rows = [prompt | chosen | prompt[-1] | rejected] per FT request (the GPU path's rows: the prompt
    once for both responses, same clipping to the model's positions);
  * ``SampledTickCPU.run`` executes ``rows`` of them, drawn proportionally from the three kinds (at least one
    of every kind present, evenly spaced inside each kind), through EVERY decoder layer of the fp32 oracle
    (OracleModel.layer: same norms / projections / RoPE / GQA / MLP as the oracle), each row attending over
    its real causal context length (prefill / fine-tune row at position t: t + 1 keys; decode row: the prompt
    plus its decode window). KV values come from a fixed synthetic pool -- the cost of a row does not depend
    on the values in its context. Decode rows end in the tied lm_head + argmax, fine-tune rows predicting a
    response token in lm_head + log-softmax; the DPO backward of fine-tune rows is NOT sampled (this flatters
    the CPU, which keeps the reported GPU/CPU ratio conservative).
Throughput = sampled rows / seconds of this execution (tokens/s: one row is one hybrid-iteration token).
"""
from __future__ import annotations

import math
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from oracle.model_ref import OracleModel

KIND_PREFILL, KIND_DECODE, KIND_FT = 0, 1, 2


def composition(engine, plan, max_pos: int) -> dict:
    """Rows of the bin the reference is about to execute (call from an Engine._execute override BEFORE
    super()._execute). Each row: (kind, position, context keys, predicts a token)."""
    from macesim.workload import WorkloadType

    rows: list[tuple[int, int, int, bool]] = []
    n_pre = n_dec = n_ft = 0
    for r in plan.bin.tasks:
        P = len(r.prompt_tokens)
        if r.workload is WorkloadType.PREFILL:
            shared = engine.trie.cached_prefix_len(r.prompt_tokens) if engine.trie is not None else 0
            for t in range(shared, P):
                rows.append((KIND_PREFILL, t, t + 1, False))
            n_pre += P - shared
        elif r.workload is WorkloadType.DECODE:
            k = r.decode_pos
            rows.append((KIND_DECODE, P - 1 + k, P + k, True))
            n_dec += 1
        else:
            room = max(1, max_pos - P)
            n_c, n_r = min(r.pair.tokens_chosen, room), min(r.pair.tokens_rejected, room)
            # the GPU path's pair layout [prompt | chosen | prompt[-1] | rejected] (engine.build_batch): prompt rows
            # once, the chosen branch, then the rejected branch re-entering at position P-1 (keys: prompt[:-1] +
            # its own rows)
            for t in range(P + n_c):
                rows.append((KIND_FT, t, t + 1, P - 1 <= t < P - 1 + n_c))
            for i in range(n_r + 1):
                rows.append((KIND_FT, P - 1 + i, P + i, i < n_r))
            n_ft += P + n_c + 1 + n_r
    return {"rows": rows, "n_prefill": n_pre, "n_decode": n_dec, "n_ft": n_ft}


def sample_rows(comp: dict, n: int) -> list[tuple[int, int, int, bool]]:
    """n rows drawn proportionally from the kinds (>= 1 per present kind), evenly spaced within each kind."""
    by = {k: [r for r in comp["rows"] if r[0] == k] for k in (KIND_PREFILL, KIND_DECODE, KIND_FT)}
    total = sum(len(v) for v in by.values())
    if total <= n:
        return list(comp["rows"])
    out = []
    for k, rs in by.items():
        if not rs:
            continue
        m = max(1, int(round(n * len(rs) / total)))
        idx = np.linspace(0, len(rs) - 1, m).round().astype(int)
        out += [rs[i] for i in idx]
    return out


def host_weights(cfg, seed: int = 0, threads: int | None = None) -> dict[str, torch.Tensor]:
    """Seeded random-init weights for the CPU arm, bf16-rounded then fp32 (the oracle's numerics), generated
    in parallel with one generator per tensor (CPU and CUDA generators differ anyway; the values do not
    change the cost of a row)."""
    names = list(cfg.param_shapes().items())
    resid_std = cfg.init_std / math.sqrt(2 * cfg.n_layers)

    def make(i_ns):
        i, (name, shape) = i_ns
        g = torch.Generator().manual_seed(seed * 100003 + i)
        t = torch.randn(shape, generator=g)
        if name == "embed":
            t *= cfg.embed_std
        elif name == "pos_embed":
            t *= 0.01
        elif name.endswith("norm.w"):
            t = 1.0 + 0.05 * t
        elif name.endswith(".b"):
            t *= 0.02
        elif name.endswith("o.w") or name.endswith("down.w"):
            t *= resid_std
        else:
            t *= cfg.init_std
        return name, t.to(torch.bfloat16).float()

    with ThreadPoolExecutor(max_workers=threads or torch.get_num_threads()) as ex:
        return dict(ex.map(make, enumerate(names)))


class SampledTickCPU:
    def __init__(self, cfg, weights_f32: dict[str, torch.Tensor], seed: int = 0):
        self.cfg = cfg
        self.model = OracleModel.__new__(OracleModel)  # adopt the fp32 weights without another copy
        self.model.cfg = cfg
        self.model.dev = torch.device("cpu")
        self.model.w = weights_f32
        g = torch.Generator().manual_seed(seed)
        n_ctx = cfg.max_pos + 1024
        self.K = torch.randn(n_ctx, cfg.n_kv_heads, cfg.head_dim, generator=g) * 0.5  # synthetic context pool
        self.V = torch.randn(n_ctx, cfg.n_kv_heads, cfg.head_dim, generator=g) * 0.5

    @torch.no_grad()
    def run(self, rows: list[tuple[int, int, int, bool]]) -> float:
        """Execute the rows; returns seconds."""
        c = self.cfg
        if not rows:
            return 0.0
        t0 = time.perf_counter()
        pos = [r[1] for r in rows]
        ctx = [min(r[2], self.K.shape[0]) for r in rows]
        x = self.model.embed([(7 * i + 11) % c.vocab for i in range(len(rows))], pos)

        def attend(l, q, k, v):
            o = torch.empty(q.shape[0], c.n_heads, c.head_dim)
            for i, n in enumerate(ctx):  # the row's own key counts the latest key (written this layer)
                K = torch.cat([self.K[: n - 1], k[i: i + 1]])
                V = torch.cat([self.V[: n - 1], v[i: i + 1]])
                mask = torch.ones(1, c.n_kv_heads, n, dtype=torch.bool)
                o[i: i + 1] = self.model.attention(q[i: i + 1], K, V, mask)
            return o

        for l in range(c.n_layers):
            x = self.model.layer(l, x, pos, attend)
        head = [i for i, r in enumerate(rows) if r[3]]
        if head:
            logits = self.model.final(x[head])
            kinds = torch.tensor([rows[i][0] for i in head])
            if (kinds == KIND_DECODE).any():
                logits[kinds == KIND_DECODE].argmax(-1)
            if (kinds == KIND_FT).any():
                torch.log_softmax(logits[kinds == KIND_FT], -1)
        return time.perf_counter() - t0
