"""CPU reference arm (test/bench infrastructure only; see oracle/model_ref.py header).

The UNMODIFIED reference engine (macesim.engine.Engine) decides every bin; this subclass executes
each bin's rows with the fp32 CPU oracle (OracleExecutor) before handing the bin to the reference's
own bookkeeping (super()._execute). None of the product's kernels, model runner or GpuEngine is on
this path. Used by ``bench.py --impl reference`` and bench.py's ``cpu_baseline`` leg.

Per-request KV (no trie page sharing): prefill computes the whole prompt; the throughput count uses
the same "hybrid-iteration tokens" definition as the GPU arm (effective prefill tokens as the
reference charges them + decode tokens + fine-tune tokens), so the CPU path is, if anything,
charged for work it did in excess.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.model_ref import OracleExecutor


def _pair_tokens(seed, rid, n_c, n_r, vocab):
    c = np.random.default_rng([seed, 307, rid]).integers(0, vocab, n_c).tolist()
    r = np.random.default_rng([seed, 308, rid]).integers(0, vocab, n_r).tolist()
    return c, r


def make_reference_engine_cls():
    from macesim.engine import Engine
    from macesim.workload import WorkloadType

    class OracleEngine(Engine):
        def setup(self, cfg, weights, tcfg, selected, seed):
            self.mcfg = cfg
            self.ox = OracleExecutor(cfg, weights, tcfg, selected)
            self.seed = seed
            self.tick_tokens = []
            self.tick_secs = []
            self.last_tok: dict[int, int] = {}
            self._tick_budget = None
            self._done = 0

        def _execute(self, plan):
            import time

            t0 = time.perf_counter()
            tasks = plan.bin.tasks
            pre = [r for r in tasks if r.workload is WorkloadType.PREFILL]
            dec = sorted((r for r in tasks if r.workload is WorkloadType.DECODE), key=lambda r: r.id)
            fts = sorted((r for r in tasks if r.workload is WorkloadType.FINETUNE), key=lambda r: r.id)
            n_tok = 0
            with torch.no_grad():
                for r in pre:
                    shared = self.trie.cached_prefix_len(r.prompt_tokens) if self.trie is not None else 0
                    self.ox.prefill(r.id, r.prompt_tokens)
                    n_tok += len(r.prompt_tokens) - shared
                for r in dec:
                    x = r.prompt_tokens[-1] if r.decode_pos == 0 else self.last_tok[r.id]
                    kept = list(self.state[r.id].kept) if self.pruning and self.state[r.id].kept else None
                    logits = self.ox.decode(r.id, x, kept)
                    self.last_tok[r.id] = int(logits.argmax())
                    n_tok += 1
            if fts:
                pairs = []
                for r in fts:
                    P = len(r.prompt_tokens)
                    room = max(1, self.mcfg.max_pos - P)
                    n_c, n_r = min(r.pair.tokens_chosen, room), min(r.pair.tokens_rejected, room)
                    if getattr(r.pair, "chosen", None):  # trace v2 content
                        c, j = list(r.pair.chosen[:n_c]), list(r.pair.rejected[:n_r])
                    else:
                        c, j = _pair_tokens(self.seed, r.id, n_c, n_r, self.mcfg.vocab)
                    pairs.append((r.id, r.prompt_tokens, c, j))
                    n_tok += 2 * P + len(c) + len(j)
                _, _, grads = self.ox.dpo_step(pairs)
                self.ox.adamw(grads)
            self.tick_secs.append(time.perf_counter() - t0)
            self.tick_tokens.append(n_tok)
            super()._execute(plan)
            for r in tasks:
                if self.state[r.id].retired:
                    self.ox.release(r.id)
            self._done += 1
            if self._tick_budget is not None and self._done >= self._tick_budget:
                raise StopIteration

        def run_ticks(self, n):
            self._tick_budget = self._done + n
            try:
                self.run()
            except StopIteration:
                pass
            self._tick_budget = None

    return OracleEngine
