"""Measured-cost loop: B200-measured latency / memory rows for the reference's ``calibrate``.

The reference's cost model (cost_model.py:25-73) is a linear stand-in with placeholder coefficients meant to
be "overwritten by calibration against a measured profile" (cost_model.py:28-30); ``calibrate`` fits it from a
CSV ``workload,batch_size,tokens,latency_ms,memory_mb`` (cost_model.py:140-205). This module produces that CSV
from the hybrid step itself:

  prefill   one request of n prompt tokens alone in a tick (GpuEngine, measured clock): latency = the tick's
            device time; memory = n x (KV bytes per token + the per-row activation buffers of the step)
  decode    B requests decoding together (a decode-only tick of B rows, median over its decode ticks):
            latency = the tick's device time; tokens = B new KV tokens; memory = B x KV bytes per token
  finetune  one DPO pair alone in a tick: tokens = chosen + rejected, latency = the tick's device time (pi_ref
            and policy passes, fused DPO, backward of the selected layers, masked AdamW); memory = the fine-tune
            row buffers (HybridModel.ft_bytes_per_token) x (prompt + chosen + 1 + rejected): one sequence per
            pair, the prompt rows shared by both responses (engine.build_batch)

Every point runs through the unmodified reference scheduler (GpuEngine mode "M" on a hand-built trace), so the
measured tick is exactly the bin the scheduler forms; memory is counted from the buffers the step allocates.
"""
from __future__ import annotations

import statistics
from pathlib import Path

import numpy as np

from .refpath import ensure_macesim

ensure_macesim()
from macesim.cost_model import CostProfile, calibrate  # noqa: E402
from macesim.workload import PreferencePair, Request, WorkloadType  # noqa: E402

HEADER = "workload,batch_size,tokens,latency_ms,memory_mb"
MB = float(1 << 20)


def row_bytes(cfg) -> int:
    """Activation bytes one inference row occupies in the step's buffers (HybridModel._ensure, shared rows)."""
    return (4 * cfg.d_model + 2 * cfg.d_model + 2 * cfg.qkv_dim + 2 * cfg.n_heads * cfg.head_dim + 8 * cfg.n_heads
            + 2 * cfg.up_dim + 2 * cfg.ffn)


def _prompt(rng, n, vocab):
    return rng.integers(1, vocab, n).tolist()


def _run(model, wl, trace, max_decode_batch=256):
    """Run a hand-built trace to completion in mode M; (device ms, (n_prefill_tokens, n_dec, n_ft_pairs)) per tick."""
    from dataclasses import replace

    from macesim.engine import EngineConfig
    from macesim.priority import PriorityParams

    from .engine import GpuEngine

    prof = replace(wl.profile, capacity=1e9, weights_resident=wl.profile.weights_resident)
    sched = replace(wl.sched, max_decode_batch=max_decode_batch, tau_task=max(wl.sched.tau_task, max_decode_batch))
    eng = GpuEngine(trace, prof, sched, PriorityParams(), wl.cache, wl.env(), EngineConfig(seed=wl.seed), None,
                    model=model, mode="M", page_budget=False)
    eng.keep_outputs = False
    comp = []
    orig = eng.build_batch

    def spy(pre, dec, fts):
        b = orig(pre, dec, fts)
        comp.append((b.n_prefill_tokens, b.n_dec, len(b.ft_pairs)))
        return b

    eng.build_batch = spy
    eng.run()
    return list(zip(eng.device_ms(), comp))


def measure_rows(model, wl, prefill_tokens=(128, 256, 512, 1024, 2048), decode_batches=(8, 32, 64, 128, 256),
                 decode_ctx=1024, ft_lens=((16, 16), (32, 32), (64, 64), (128, 128)), ft_prompt=512, repeats=2,
                 seed=0) -> list[tuple]:
    cfg = model.cfg
    rng = np.random.default_rng(seed)
    lim = min(model.max_prompt_len, cfg.max_pos - 8)  # prompts the model's page tables / positions can hold
    prefill_tokens = [n for n in prefill_tokens if n <= lim]
    decode_ctx = min(decode_ctx, lim)
    ft_prompt = min(ft_prompt, lim // 2)
    kv = cfg.kv_bytes_per_token()
    rows: list[tuple] = []
    rid = 0

    def req(**kw):
        nonlocal rid
        rid += 1
        return Request(id=rid, tenant=0, arrival_time=0.0, **kw)

    # one discarded warm-up of every tick kind: the first launches of a process pay one-time costs (tensor-map
    # and function-attribute set-up, allocator growth) that are not the device time of the workload
    _run(model, wl, [req(workload=WorkloadType.PREFILL, prompt_tokens=_prompt(rng, min(256, lim), cfg.vocab),
                         target_output_len=3),
                     req(workload=WorkloadType.FINETUNE, prompt_tokens=_prompt(rng, min(64, lim // 2), cfg.vocab),
                         target_output_len=8, pair=PreferencePair(0.5, 8, 8))])

    for _ in range(repeats):
        for n in prefill_tokens:  # prefill alone in its tick
            out = _run(model, wl, [req(workload=WorkloadType.PREFILL, prompt_tokens=_prompt(rng, n, cfg.vocab),
                                       target_output_len=1)])
            ms = [t for t, (p, d, f) in out if p == n and d == 0 and f == 0]
            rows.append(("prefill", 1, n, ms[0], n * (kv + row_bytes(cfg)) / MB))
        for B in decode_batches:  # B decodes together (after their prefills)
            trace = [req(workload=WorkloadType.PREFILL, prompt_tokens=_prompt(rng, decode_ctx, cfg.vocab),
                         target_output_len=6) for _ in range(B)]
            out = _run(model, wl, trace, max_decode_batch=B)
            ms = [t for t, (p, d, f) in out if p == 0 and d == B and f == 0]
            if ms:
                rows.append(("decode", B, B, statistics.median(ms), B * kv / MB))
        for c, r in ft_lens:  # one DPO pair alone in its tick
            out = _run(model, wl, [req(workload=WorkloadType.FINETUNE,
                                       prompt_tokens=_prompt(rng, ft_prompt, cfg.vocab), target_output_len=c,
                                       pair=PreferencePair(0.5, c, r))])
            ms = [t for t, (p, d, f) in out if f == 1 and p == 0 and d == 0]
            rows.append(("finetune", 1, c + r, ms[0], model.ft_bytes_per_token() * (ft_prompt + c + 1 + r) / MB))
    return rows


def write_csv(rows, path) -> None:
    Path(path).write_text(HEADER + "\n" + "".join(f"{w},{b},{t},{lat!r},{mem!r}\n" for w, b, t, lat, mem in rows))


def calibrated(path, base: CostProfile):
    """The reference's own fit (cost_model.calibrate) of the measured rows."""
    return calibrate(path, base)

