"""Vectorised host bookkeeping for the reference loop, decision-for-decision identical.

The hybrid iteration's end-to-end rate is bound by the reference's per-tick Python, not by the B200: at C2
the queue holds ~1.8k requests and every tick re-keys all of them (priority.py:121-127), and every decode
row draws its synthetic head norms through its own numpy Generator (engine.py:433-442). Both are restated
here without changing a single decision:

* ``FastPriorityQueue`` keeps the reference's key ``(-p, arrival, id)`` per queued request (priority.py:112-116)
  in column arrays; push keys a request with the reference's own ``_key``; ``refresh`` recomputes every p
  with numpy in the same IEEE-754 operation order as ``dynamic_priority`` / ``ft_total_priority``
  (priority.py:67-81: base + growth * (t - arrival), then + gamma * loss for fine-tunes) and sorts the keys
  once. Keys are unique (they contain the request id), so the pop / peek sequence equals heappop on the
  reference heap. ``priority_state`` (priority.py:114-115, written but never read by the reference) holds
  the refreshed value for every popped request.
* ``NormStream`` draws a request's head-norm jitter ``normal(1, 0.1)`` in blocks from the same Generator
  (seed ``[seed, 211, id]``); numpy's Generator fills an array with the same sequence as repeated
  ``size=num_heads`` calls, so the per-step values equal the reference's (checked in tests/test_host_cpu.py).
* ``fast_schedule_iteration`` runs Alg. 1 (scheduler.py:133-188) natively (csrc/hostsched.cu) over the queue
  head with precomputed estimates, with an inlined Python restatement for the iterations it hands back.
* ``make_bulk_pair_losses`` restates the fine-tune loss chain (alignment.py:39-47, 151-166) for many requests
  per refresh / push_many, value for value.
"""
from __future__ import annotations

import numpy as np

from .refpath import ensure_macesim

ensure_macesim()
from macesim.priority import PriorityContractError, PriorityQueue  # noqa: E402
from macesim.scheduler import Bin, TickPlan  # noqa: E402
from macesim.workload import WorkloadType  # noqa: E402

_FT = WorkloadType.FINETUNE
_DEC = WorkloadType.DECODE


class FastPriorityQueue(PriorityQueue):
    """The reference PriorityQueue's semantics on column arrays: a key (-p, arrival, id) per live entry, computed
    by the reference's own ``_key`` at push time (priority.py:112-119) and re-computed for all entries by a
    vectorised ``refresh``; ``pop`` / ``peek`` return the entry with the smallest key, exactly like heappop on
    the reference heap (keys are unique: they contain the request id)."""

    def __init__(self, params, loss_fn=None):
        super().__init__(params, loss_fn)
        cap = 1024
        self._neg = np.empty(cap, np.float64)   # -p of the current key
        self._arr = np.empty(cap, np.float64)   # arrival time
        self._bg = np.empty((cap, 2), np.float64)  # base, growth of the workload type
        self._id = np.empty(cap, np.int64)
        self._ft = np.zeros(cap, bool)
        self._alive = np.zeros(cap, bool)
        self._req: list = [None] * cap
        self._n = 0          # slots used (live + dead)
        self._live = 0
        self._order: list[int] | None = None  # pop order of live slots after refresh (None: stale)
        self._cur = 0
        # id -> (arrival, base, growth, is fine-tune, workload): a prefill turns into a decode in place
        # (workload.py:64-66), so an entry is only reused while the request's workload is unchanged
        self._meta: dict[int, tuple] = {}
        self.bulk_loss = None          # optional many-request loss_fn (make_bulk_pair_losses)
        # pushed keys not yet in the columns: (-p, arrival, base, growth, id, is fine-tune, request)
        self._pend: list[tuple] = []
        self._popped = False  # any pop since the last sort

    def _meta_of(self, req) -> tuple:
        w = req.workload
        m = (req.arrival_time, self.params.base[w], self.params.growth[w], w is _FT, w)
        self._meta[req.id] = m
        return m

    def __len__(self) -> int:
        return self._live

    def __bool__(self) -> bool:
        return self._live > 0

    def _grow(self) -> None:
        cap = 2 * self._neg.shape[0]
        for name in ("_neg", "_arr", "_id", "_ft", "_alive"):
            a = getattr(self, name)
            b = np.zeros(cap, a.dtype)
            b[: a.shape[0]] = a
            setattr(self, name, b)
        bg = np.zeros((cap, 2), np.float64)
        bg[: self._bg.shape[0]] = self._bg
        self._bg = bg
        self._req += [None] * (cap - len(self._req))

    def _compact(self) -> None:
        idx = np.flatnonzero(self._alive[: self._n])
        n = idx.shape[0]
        for name in ("_neg", "_arr", "_id", "_ft", "_alive"):
            a = getattr(self, name)
            a[:n] = a[idx]
        self._bg[:n] = self._bg[idx]
        reqs = [self._req[i] for i in idx.tolist()]
        self._req[:n] = reqs
        for k in range(n, self._n):
            self._req[k] = None
        self._alive[n: self._n] = False
        self._n = n
        self._order = None

    def push(self, req, t=None) -> None:  # priority.py:118-119 (key of _key / priority_of, same arithmetic)
        t = self._last_refresh if t is None else t
        m = self._meta.get(req.id)
        if m is None or m[4] is not req.workload:
            m = self._meta_of(req)
        arrival, base, growth, is_ft, _ = m
        if t < arrival:
            raise PriorityContractError(
                f"priority query at t={t} before arrival of request {req.id} at {arrival}")
        p = base + growth * (t - arrival)  # dynamic_priority (priority.py:73)
        if is_ft and self.loss_fn is not None:  # ft_total_priority (priority.py:76-81)
            loss = self.loss_fn(req) if self.bulk_loss is None else self.bulk_loss((req,))[0]
            if loss < 0:
                raise PriorityContractError("loss must be >= 0 under the positive-loss convention")
            p = p + self.params.gamma * loss
        ps = req.priority_state
        ps.value = p
        ps.refreshed_at = t
        # keys land in the columns in bulk at the next refresh / pop / peek (_flush)
        self._pend.append((-p, arrival, base, growth, req.id, is_ft, req))
        self._live += 1
        self._order = None

    def push_many(self, reqs, t: float) -> None:
        """push(req, t) for every request, keys computed together (same arithmetic, same contract checks)."""
        n = len(reqs)
        if not n:
            return
        meta = self._meta
        ms = []
        for r in reqs:
            m = meta.get(r.id)
            if m is None or m[4] is not r.workload:
                m = self._meta_of(r)
            ms.append(m)
        arr = np.fromiter((m[0] for m in ms), np.float64, n)
        if (t < arr).any():
            bad = reqs[int(np.argmax(t < arr))]
            raise PriorityContractError(
                f"priority query at t={t} before arrival of request {bad.id} at {bad.arrival_time}")
        base = np.fromiter((m[1] for m in ms), np.float64, n)
        growth = np.fromiter((m[2] for m in ms), np.float64, n)
        p = base + growth * (t - arr)  # dynamic_priority (priority.py:73), elementwise, no FMA
        fts = [i for i, m in enumerate(ms) if m[3]]
        if fts and self.loss_fn is not None:  # ft_total_priority (priority.py:76-81)
            fr = [reqs[i] for i in fts]
            losses = self.bulk_loss(fr) if self.bulk_loss is not None else [self.loss_fn(r) for r in fr]
            gamma = self.params.gamma
            for i, loss in zip(fts, losses):
                if loss < 0:
                    raise PriorityContractError("loss must be >= 0 under the positive-loss convention")
                p[i] = p[i] + gamma * loss
        pl = p.tolist()
        for r, v in zip(reqs, pl):
            ps = r.priority_state
            ps.value = v
            ps.refreshed_at = t
        # straight into the columns (no pending tuples)
        self._reserve(n, len(self._pend))
        k0, k1 = self._n, self._n + n
        self._neg[k0:k1] = -p
        self._arr[k0:k1] = arr
        self._bg[k0:k1, 0] = base
        self._bg[k0:k1, 1] = growth
        self._id[k0:k1] = [r.id for r in reqs]
        self._ft[k0:k1] = [m[3] for m in ms]
        self._alive[k0:k1] = True
        self._req[k0:k1] = reqs
        self._n = k1
        self._live += n
        self._order = None

    def _reserve(self, n_new: int, pending: int = 0) -> None:
        """Room for n_new more column entries (``pending``: how many of the live count are not in the columns)."""
        while self._n + n_new > self._neg.shape[0]:
            if self._live - pending < self._n // 2:
                self._compact()
                if self._n + n_new <= self._neg.shape[0]:
                    break
            self._grow()

    def _flush(self) -> None:
        n_new = len(self._pend)
        if not n_new:
            return
        self._reserve(n_new, n_new)
        k0, k1 = self._n, self._n + n_new
        pn, pa, pb, pg, pi, pf, preq = zip(*self._pend)
        self._neg[k0:k1] = pn
        self._arr[k0:k1] = pa
        self._bg[k0:k1, 0] = pb
        self._bg[k0:k1, 1] = pg
        self._id[k0:k1] = pi
        self._ft[k0:k1] = pf
        self._alive[k0:k1] = True
        self._req[k0:k1] = preq
        self._n = k1
        self._pend = []

    def refresh(self, t: float) -> None:  # priority.py:121-127
        self._last_refresh = t
        if self._live == 0:
            return
        self._flush()
        if self._live < self._n // 2:
            self._compact()
        n = self._n
        alive = self._alive[:n]
        arr = self._arr[:n]
        if ((t < arr) & alive).any():
            bad = self._req[int(np.argmax((t < arr) & alive))]
            raise PriorityContractError(
                f"priority query at t={t} before arrival of request {bad.id} at {bad.arrival_time}")
        p = self._bg[:n, 0] + self._bg[:n, 1] * (t - arr)  # dynamic_priority (priority.py:73), no FMA
        if self.loss_fn is not None:
            gamma = self.params.gamma
            ks = np.flatnonzero(self._ft[:n] & alive).tolist()
            reqs = self._req
            losses = (self.bulk_loss([reqs[k] for k in ks]) if self.bulk_loss is not None
                      else [self.loss_fn(reqs[k]) for k in ks])
            for k, loss in zip(ks, losses):  # ft_total_priority (priority.py:76-81)
                if loss < 0:
                    raise PriorityContractError("loss must be >= 0 under the positive-loss convention")
                p[k] = p[k] + gamma * loss
        self._neg[:n] = -p
        self._sort()

    def _sort(self) -> None:
        n = self._n
        live = np.flatnonzero(self._alive[:n])
        o = np.lexsort((self._id[live], self._arr[live], self._neg[live]))  # heappop order of (-p, arrival, id)
        self._order = live[o].tolist()
        self._cur = 0
        self._popped = False

    def _front(self) -> int:
        if self._live == 0:
            raise IndexError("pop from empty priority queue")
        if self._order is None:
            self._flush()
            self._sort()
        while not self._alive[self._order[self._cur]]:
            self._cur += 1
        return self._order[self._cur]

    def pop(self):
        k = self._front()
        self._popped = True
        self._alive[k] = False
        self._live -= 1
        self._cur += 1
        req = self._req[k]
        self._req[k] = None
        req.priority_state.value = -float(self._neg[k])
        req.priority_state.refreshed_at = self._last_refresh
        return req

    def head(self, K: int) -> list[int] | None:
        """Slots of the first K entries in pop order, when nothing was popped since the last sort (then
        every entry of the order is live); None otherwise."""
        if self._order is None:
            self._flush()
            self._sort()
        if self._popped:
            return None
        return self._order[self._cur: self._cur + K]

    def pop_head(self, ks: list[int]) -> None:
        """Pop the entries ``head`` returned (a prefix of it), as that many pop() calls would."""
        m = len(ks)
        if not m:
            return
        self._alive[ks] = False
        self._live -= m
        self._cur += m
        self._popped = True
        t = self._last_refresh
        reqs = self._req
        for k, v in zip(ks, (-self._neg[ks]).tolist()):
            ps = reqs[k].priority_state
            ps.value = v
            ps.refreshed_at = t
            reqs[k] = None

    def peek(self):
        if self._order is not None or self._live == 0:
            return self._req[self._front()]
        # keys changed since the last sort (pushes): the smallest (-p, arrival, id) without sorting
        self._flush()
        idx = np.flatnonzero(self._alive[: self._n])
        neg = self._neg[idx]
        c = idx[neg == neg.min()]
        if c.shape[0] > 1:
            arr = self._arr[c]
            c = c[arr == arr.min()]
            if c.shape[0] > 1:
                c = c[np.argmin(self._id[c]):][:1]
        return self._req[int(c[0])]


def make_bulk_pair_losses(env):
    """pair_loss for many fine-tune requests at once, value-for-value equal to the reference chain
    Engine._loss_of -> AlignmentEnv.pair_loss -> pair_margin -> dpo_loss (alignment.py:39-47, 151-166): the
    per-request offset initial_margin - (mu0 - drift_rate * arrival) is computed once with the reference's
    arithmetic, margin = mu + offset, MarginSample(margin, 0).margin = margin - 0.0, then the same math.exp /
    math.log1p branch. None when env's methods are not the reference's (a subclass may override them)."""
    import math

    from macesim.alignment import AlignmentEnv

    if type(env).pair_loss is not AlignmentEnv.pair_loss or type(env).pair_margin is not AlignmentEnv.pair_margin:
        return None
    offs: dict[int, float] = {}
    exp, log1p = math.exp, math.log1p
    tenants = env.tenants

    def losses(reqs) -> list[float]:
        beta = env.beta
        if beta <= 0:  # dpo_loss raises AlignmentDomainError: let the reference say so
            return [env.pair_loss(r) for r in reqs]
        out = []
        for r in reqs:
            o = offs.get(r.id)
            if o is None:
                env.pair_margin(r)  # the reference's own argument checks (workload / pair / tenant)
                prm = tenants[r.tenant].params
                o = offs[r.id] = r.pair.initial_margin - (prm.mu0 - prm.drift_rate * r.arrival_time)
            x = -beta * ((tenants[r.tenant].mu + o) - 0.0)
            out.append(x + log1p(exp(-x)) if x > 0 else log1p(exp(x)))
        return out

    return losses


class NormStream:
    """Per-request synthetic head-norm jitter in blocks (engine.py:433-442), stored per KV slot so a tick's
    decode rows are served by one gather; only rows whose block ran out draw from their Generator."""

    BLOCK = 64  # steps per draw

    def __init__(self, engine, n_slots: int):
        self.eng = engine
        H = engine.cache_cfg.num_heads
        self.blk = np.zeros((n_slots, self.BLOCK, H))
        self.cur = np.zeros(n_slots, np.int64)
        self.owner = np.full(n_slots, -1, np.int64)  # request id whose block the slot holds

    def _refill(self, req, rs, slot: int) -> None:
        eng = self.eng
        H = eng.cache_cfg.num_heads
        if rs.head_rng is None:
            rs.head_rng = np.random.default_rng([eng.ecfg.seed, 211, req.id])
            rs.head_scales = [eng.cache_cfg.weak_scale if h in eng.weak_heads else 1.0 for h in range(H)]
        block = rs.head_rng.normal(1.0, 0.1, size=H * self.BLOCK).reshape(self.BLOCK, H)
        self.blk[slot] = np.maximum(0.0, np.asarray(rs.head_scales, np.float64) * block)
        self.cur[slot] = 0
        self.owner[slot] = req.id

    def norms(self, req, rs) -> np.ndarray:
        slot = self.eng.slot_of[req.id]
        if self.owner[slot] != req.id or self.cur[slot] >= self.BLOCK:
            self._refill(req, rs, slot)
        c = int(self.cur[slot])
        self.cur[slot] = c + 1
        return self.blk[slot, c].copy()

    def norms_many(self, rows, slots: np.ndarray) -> np.ndarray:
        """[n, H] norms of this step for decode rows ``rows`` in KV slots ``slots`` (distinct)."""
        ids = np.fromiter((r.id for r in rows), np.int64, len(rows))
        state = self.eng.state
        for i in np.flatnonzero((self.owner[slots] != ids) | (self.cur[slots] >= self.BLOCK)).tolist():
            r = rows[i]
            self._refill(r, state[r.id], int(slots[i]))
        c = self.cur[slots]
        self.cur[slots] = c + 1
        return self.blk[slots, c]

    def drop(self, rid: int) -> None:
        slot = self.eng.slot_of.get(rid)
        if slot is not None and self.owner[slot] == rid:
            self.owner[slot] = -1


def _native_alg1(queue, capacity_budget, cfg, estimator, hard_limit, dec_est):
    """Alg. 1 over the queue's head with csrc/hostsched.cu (mace_host_alg1); None hands the iteration to the
    Python loop (something was popped since the sort, or the dequeue would run past tau_task candidates)."""
    K = min(len(queue), cfg.tau_task)
    ks = queue.head(K)
    if ks is None or not ks:
        return None
    reqs = [queue._req[k] for k in ks]
    DEC, FT = _DEC, _FT
    try:
        ests = [dec_est if (dec_est is not None and r.workload is DEC) else estimator(r) for r in reqs]
    except Exception:  # e.g. a malformed request past the stop point: the Python loop raises where Alg. 1 would
        return None
    n = len(reqs)
    mem = np.array([e.mem for e in ests], np.float64)
    lat = np.array([e.lat for e in ests], np.float64)
    ft = np.array([r.workload is FT for r in reqs], np.int8)
    assign = np.empty(n, np.int32)
    counts = np.zeros(5, np.int32)
    bin0 = np.zeros(2, np.float64)
    from ._lib import lib
    rc = lib().mace_host_alg1(n, mem.ctypes.data, lat.ctypes.data, ft.ctypes.data, int(len(queue) > n),
                              float(capacity_budget), float(hard_limit), float(cfg.tau_mem * capacity_budget),
                              int(cfg.tau_task), float(cfg.lambda1), float(cfg.lambda2), int(cfg.max_ft_batch),
                              int(cfg.max_decode_batch), assign.ctypes.data, counts.ctypes.data, bin0.ctypes.data)
    if rc == 2:
        return None
    if rc != 0:
        raise RuntimeError(f"mace_host_alg1 failed ({rc})")
    count, n_bins, examined = int(counts[0]), int(counts[1]), int(counts[2])
    queue.pop_head(ks[:count])
    plan = TickPlan(bin=Bin(capacity_budget))
    plan.dequeued.extend(reqs[:count])
    tasks = [[] for _ in range(n_bins)]
    estl = [[] for _ in range(n_bins)]
    deferred = []
    for r, e, a in zip(reqs[:count], ests[:count], assign[:count].tolist()):
        if a >= 0:
            tasks[a].append(r)
            estl[a].append(e)
        elif a == -1:
            plan.rejected.append(r)
        else:
            deferred.append(r)
    plan.bins_opened += n_bins
    plan.bins_examined = examined
    if n_bins:
        plan.bin = Bin(capacity_budget, tasks=tasks[0], estimates=estl[0], used_memory=float(bin0[0]),
                       max_latency=float(bin0[1]), n_inference=int(counts[3]), n_ft=int(counts[4]))
        for later in tasks[1:]:
            plan.requeued.extend(later)
    plan.requeued.extend(deferred)
    return plan


def fast_schedule_iteration(queue, capacity_budget, cfg, estimator, t, hard_limit=None, dec_est=None,
                            native=True):
    """Alg. 1 exactly as scheduler.py:133-188 (same dequeue stop rule, same best-fit score arithmetic
    lambda1*|free - mem| + lambda2*|maxlat - lat| with free = budget - used, same strict '<' tie rule,
    same requeue / defer / reject lists), with the Bin methods (scheduler.py:81-117) inlined into local
    arithmetic. Returns the reference TickPlan / Bin types; tests/test_host_cpu.py checks plan-for-plan
    equality against the reference on randomized queues. ``dec_est``: the estimator's (constant) decode
    estimate (cost_model.py:100-102), used without the call when given."""
    if hard_limit is None:
        hard_limit = capacity_budget
    if native and isinstance(queue, FastPriorityQueue) and len(queue):
        plan = _native_alg1(queue, capacity_budget, cfg, estimator, hard_limit, dec_est)
        if plan is not None:
            return plan
    plan = TickPlan(bin=Bin(capacity_budget))
    FT = _FT
    max_ft, max_inf = cfg.max_ft_batch, cfg.max_decode_batch
    l1, l2 = cfg.lambda1, cfg.lambda2
    stop_mem = cfg.tau_mem * capacity_budget
    tau_task = cfg.tau_task
    # bin state: [used, maxlat, n_inf, n_ft, tasks, ests]
    bins: list[list] = []
    deferred: list = []
    dequeued = plan.dequeued
    rejected = plan.rejected
    examined = 0
    count = 0
    pop = queue.pop
    DEC = _DEC
    while queue:
        if bins and (bins[0][0] >= stop_mem or count >= tau_task):
            break
        task = pop()
        count += 1
        dequeued.append(task)
        est = dec_est if (dec_est is not None and task.workload is DEC) else estimator(task)
        mem, lat = est.mem, est.lat
        if mem > hard_limit:
            rejected.append(task)
            continue
        if mem > capacity_budget:
            deferred.append(task)
            continue
        is_ft = task.workload is FT
        best = None
        best_score = float("inf")
        for b in bins:
            examined += 1
            free = capacity_budget - b[0]
            if free < mem:
                continue
            if (b[3] < max_ft) if is_ft else (b[2] < max_inf):
                score = l1 * abs(free - mem) + l2 * abs(b[1] - lat)
                if score < best_score:
                    best_score = score
                    best = b
        if best is None:
            best = [0.0, 0.0, 0, 0, [], []]
            bins.append(best)
            plan.bins_opened += 1
        best[4].append(task)
        best[5].append(est)
        best[0] += mem
        best[1] = max(best[1], lat)
        if is_ft:
            best[3] += 1
        else:
            best[2] += 1
    plan.bins_examined = examined
    if bins:
        b0 = bins[0]
        plan.bin = Bin(capacity_budget, tasks=b0[4], estimates=b0[5], used_memory=b0[0], max_latency=b0[1],
                       n_inference=b0[2], n_ft=b0[3])
        for later in bins[1:]:
            plan.requeued.extend(later[4])
    plan.requeued.extend(deferred)
    return plan
