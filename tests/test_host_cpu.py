"""Host-side logic on CPU (no GPU): the drop-in keeps the reference's decisions bit-identical, and the
KV page manager's tables always resolve to the right KV rows (incl. prefix sharing, splits,
copy-on-diverge and LRU eviction)."""
import json
from pathlib import Path

import pytest

from fakes import FakeModel

GOLD = Path(__file__).parent / "golden" / "c1_reference.json"


def _engine(wl, fast_host=True, **kw):
    from paper_2510_03283_b200.engine import GpuEngine

    fm = FakeModel(wl.model, wl.train, max_prompt_len=wl.max_prompt_len, **kw)
    eng = GpuEngine(*wl.engine_args(), model=fm, mode="P", fast_host=fast_host)
    eng.keep_outputs = False
    return eng, fm


def _check_tables(eng, fm):
    """Every paged sequence of the last batch reads its own prompt tokens at positions [0, n_pv)."""
    b = fm.last_batch
    slot_req = {s: r for r, s in eng.slot_of.items()}
    for s in b.seqs.tolist():
        kind, q0, ql, slot, n_pv = s[:5]
        if kind == 2:
            continue
        rid = slot_req.get(slot)
        if rid is None:  # retired inside this tick
            continue
        req = eng.trace_by_id[rid]
        view = fm.prompt_view(slot, n_pv)
        want = [(t, p) for p, t in enumerate(req.prompt_tokens[:n_pv])]
        assert view == want, f"request {rid}: page table does not resolve to its prompt"


def test_c1_timeline_identical_with_fake_device():
    from paper_2510_03283_b200.workloads import c1

    eng, fm = _engine(c1())
    eng.trace_by_id = {r.id: r for r in eng.trace}
    orig = fm.step

    def step(batch, trim=None, ft_global=None):
        out = orig(batch, trim, ft_global)
        _check_tables(eng, fm)
        return out

    fm.step = step
    res = eng.run()
    gold = json.loads(GOLD.read_text())
    assert json.loads(json.dumps(res.timeline, sort_keys=True)) == gold["timeline"]
    assert res.metrics.decoded_tokens == 442
    assert not fm.violations
    # after the trace drains only trie-owned groups stay referenced
    trie_groups = {g for pages in eng.trie.node_pages.values() for g in pages.values()}
    assert set(int(g) for g in (eng.pool.ref > 0).nonzero()[0]) == trie_groups
    assert not eng.table_of and not eng.slot_of


def test_prefix_sharing_splits_and_lru_eviction():
    """Tight capacity forces LRU offload (cache.py:217-238) while deep template trees force splits and
    copy-on-diverge pages; tables must stay correct and groups must never leak."""
    import dataclasses

    from macesim.cost_model import CostProfile
    from macesim.distributions import parse_dist
    from macesim.workload import PrefixTreeSpec
    from paper_2510_03283_b200.workloads import c1

    wl = c1(seed=3)
    tc = dataclasses.replace(wl.trace_cfg, arrival_rate=40, duration=4, retrain_rate=0.1,
                             prefix_tree_spec=PrefixTreeSpec(branching=3, depth=4,
                                                              segment_len=parse_dist("uniform:lo=5,hi=23")))
    wl = dataclasses.replace(wl, trace_cfg=tc, profile=CostProfile(capacity=14600.0, weights_resident=14000.0))
    eng, fm = _engine(wl, prompt_groups=8192)
    eng.trace_by_id = {r.id: r for r in eng.trace}
    orig = fm.step
    n_checks = [0]

    def step(batch, trim=None, ft_global=None):
        out = orig(batch, trim, ft_global)
        _check_tables(eng, fm)
        n_checks[0] += 1
        return out

    fm.step = step
    res = eng.run()
    evicts = [e for e in res.timeline if e.get("kind") == "cache_event" and e.get("event") == "evict"]
    copies = sum(c[1].page_copies.shape[0] for c in fm.calls if c[0] == "step")
    assert evicts, "config must exercise LRU eviction"
    assert copies > 0, "config must exercise copy-on-diverge"
    assert n_checks[0] == res.metrics.total_iterations
    trie_groups = {g for pages in eng.trie.node_pages.values() for g in pages.values()}
    assert set(int(g) for g in (eng.pool.ref > 0).nonzero()[0]) == trie_groups


@pytest.mark.parametrize("policy", ["Hybrid", "HybridNoPrefix", "HybridNoPrune", "Periodic", "Sync", "HybridNoBin",
                                    "NoRetrain"])
def test_baseline_policies_share_execute(policy):
    """Every policy shares _execute: the drop-in runs them unchanged and the
    timeline equals an unmodified reference run."""
    import dataclasses

    from macesim.engine import Engine
    from macesim.scheduler import Policy
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    wl = dataclasses.replace(wl, sched=dataclasses.replace(wl.sched, policy=Policy(policy)))
    ref = Engine(*wl.engine_args()).run()
    eng, fm = _engine(wl)
    res = eng.run()
    assert json.dumps(res.timeline, sort_keys=True) == json.dumps(ref.timeline, sort_keys=True)
    assert not fm.violations


def test_path_dfs_order_matches_reference():
    """The engine's O(path) DFS ordering equals the reference's whole-trie dfs_order on real tries."""
    import random

    from macesim.cache import PrefixTrie, dfs_order
    from macesim.workload import Request, WorkloadType
    from paper_2510_03283_b200.engine import path_dfs_order

    rnd = random.Random(0)
    for trial in range(30):
        trie = PrefixTrie(0.1)
        reqs = []
        base = [rnd.randrange(6) for _ in range(12)]
        for i in range(rnd.randrange(2, 25)):
            cut = rnd.randrange(0, 12)
            prompt = base[:cut] + [rnd.randrange(6) for _ in range(rnd.randrange(1, 8))]
            r = Request(id=i, tenant=0, workload=WorkloadType.PREFILL, arrival_time=0.0, prompt_tokens=prompt,
                        target_output_len=1)
            reqs.append((r, trie.insert(prompt, 0.0).leaf))
        sub = rnd.sample(reqs, rnd.randrange(2, len(reqs) + 1))
        assert [r.id for r in path_dfs_order(sub)] == [r.id for r in dfs_order(trie, sub)]


@pytest.mark.parametrize("wl_name,ticks", [("c1", None), ("c2", 260)])
def test_batched_head_stats_bit_identical(wl_name, ticks):
    """The host fast paths (hoststats.py batched head-stats/prune, hostfast.py column priority queue and
    block-drawn head norms) reproduce the reference's per-row _exec_decode and PriorityQueue exactly: same
    timeline (decisions, prune events with MB deltas), kept[] and metrics."""
    from paper_2510_03283_b200.workloads import WORKLOADS

    def run(fast):
        wl = WORKLOADS[wl_name]()
        eng, fm = _engine(wl, fast_host=fast, prompt_groups=1 << 15, max_slots=1024)
        if ticks is None:
            res = eng.run()
            return res.timeline, res.metrics.tbt_ms, {k: list(v.kept) for k, v in eng.state.items()}
        eng.run_ticks(ticks)
        return eng.timeline, eng.metrics.tbt_ms, {k: list(v.kept) for k, v in eng.state.items()}

    a, b = run(True), run(False)
    assert json.dumps(a[0], sort_keys=True) == json.dumps(b[0], sort_keys=True)
    assert a[1] == b[1]
    assert a[2] == b[2]
    assert any(e.get("event") == "prune" for e in a[0])


def test_batched_allocate_matches_reference_fuzz():
    import numpy as np

    from macesim.cache import allocate_capacity
    from paper_2510_03283_b200.hoststats import BatchedHeadStats

    rng = np.random.default_rng(0)
    # c_total >= 1024 and H up to 64: the zero-cap donor choice compares tuple fields, no digit packing
    for H, C in ((8, 160), (12, 160), (4, 10), (3, 7), (8, 4096), (64, 2048), (16, 1500)):
        hs = BatchedHeadStats(1, H, 4, C, 128, None)
        means = rng.random((4000, H)) * rng.choice([1.0, 0.01, 1e-5], size=(4000, H))
        means[rng.random((4000, H)) < 0.1] = 0.0
        means[:5] = 0.0
        got = hs._allocate(means)
        want = np.array([allocate_capacity(m.tolist(), C) for m in means])
        assert (got == want).all()


def test_fast_priority_queue_matches_reference_heap():
    """FastPriorityQueue pops in exactly the reference heap's order under interleaved push / refresh / pop /
    peek, including fine-tune keys with a loss term and equal priorities (arrival / id tie-breaks)."""
    import numpy as np

    from macesim.priority import PriorityParams, PriorityQueue
    from macesim.workload import PreferencePair, Request, WorkloadType
    from paper_2510_03283_b200.hostfast import FastPriorityQueue

    rng = np.random.default_rng(3)
    kinds = [WorkloadType.PREFILL, WorkloadType.DECODE, WorkloadType.FINETUNE]
    losses = {}

    def loss_fn(r):
        return losses[r.id]

    ref, fast = PriorityQueue(PriorityParams(), loss_fn), FastPriorityQueue(PriorityParams(), loss_fn)
    t, rid = 0.0, 0
    for step in range(300):
        batch = []
        for _ in range(int(rng.integers(0, 12))):
            w = kinds[int(rng.integers(0, 3))]
            arr = t if rng.random() < 0.3 else min(t, round(t - rng.random(), 1))  # ties on arrival time
            pair = PreferencePair(0.5, 4, 4) if w is WorkloadType.FINETUNE else None
            mk = lambda: Request(id=rid, tenant=0, workload=w, arrival_time=max(0.0, arr), prompt_tokens=[1, 2],
                                 target_output_len=4, pair=pair)
            losses[rid] = float(rng.choice([0.0, 0.3, rng.random()]))
            ref.push(mk(), t)
            batch.append(mk())
            rid += 1
        if rng.random() < 0.5:
            fast.push_many(batch, t)  # the bulk route-back path
        else:
            for r in batch:
                fast.push(r, t)
        if rng.random() < 0.5:
            t += float(rng.choice([0.0, 0.05, rng.random()]))
            for k in list(losses):
                losses[k] = float(rng.random())
            ref.refresh(t)
            fast.refresh(t)
        assert len(ref) == len(fast)
        if ref:
            assert ref.peek().id == fast.peek().id
        for _ in range(int(rng.integers(0, 10))):
            if not ref:
                break
            assert ref.pop().id == fast.pop().id


def test_cached_prefix_len_matches_reference():
    """GpuPrefixTrie.cached_prefix_len (slice compare + bisection) equals the reference's element loop on
    random tries with shared prefixes, partial label matches and uncached nodes."""
    import numpy as np

    from macesim.cache import PrefixTrie
    from paper_2510_03283_b200.kvmanager import GpuPrefixTrie, GroupPool, _common_prefix

    rng = np.random.default_rng(7)
    for _ in range(2000):
        a = rng.integers(0, 5, int(rng.integers(1, 80))).tolist()
        b = a[: int(rng.integers(0, len(a) + 1))] + rng.integers(0, 5, int(rng.integers(0, 40))).tolist()
        i = int(rng.integers(0, len(b) + 1))
        lim = min(len(a), len(b) - i)
        ref = 0
        while ref < lim and a[ref] == b[i + ref]:
            ref += 1
        assert _common_prefix(a, b, i, lim) == ref
    ref_t, gpu_t = PrefixTrie(0.1), GpuPrefixTrie(0.1, GroupPool(1))
    prompts = []
    for k in range(300):
        base = prompts[int(rng.integers(0, len(prompts)))] if prompts and rng.random() < 0.7 else []
        p = base[: int(rng.integers(0, len(base) + 1))] + rng.integers(0, 6, int(rng.integers(1, 60))).tolist()
        prompts.append(p)
        r1, r2 = ref_t.insert(p, float(k)), gpu_t.insert(p, float(k))
        if rng.random() < 0.6:  # cache the path (no pages needed for the query)
            for n in r1.leaf.path_nodes():
                n.cached = True
            for n in r2.leaf.path_nodes():
                n.cached = True
        q = prompts[int(rng.integers(0, len(prompts)))]
        q = q[: int(rng.integers(1, len(q) + 1))] + rng.integers(0, 6, int(rng.integers(0, 5))).tolist()
        assert gpu_t.cached_prefix_len(q) == ref_t.cached_prefix_len(q)


def test_fast_schedule_iteration_matches_reference():
    """hostfast.fast_schedule_iteration returns the reference Alg. 1 plan (scheduler.py:133-188) task for task on
    randomized queues: mixed workloads, tight budgets (reject / defer), bin caps, tau_mem / tau_task stops."""
    import numpy as np

    from macesim.cost_model import WorkloadEstimate
    from macesim.priority import PriorityParams, PriorityQueue
    from macesim.scheduler import SchedulerConfig, schedule_iteration
    from macesim.workload import PreferencePair, Request, WorkloadType
    from paper_2510_03283_b200.hostfast import FastPriorityQueue, fast_schedule_iteration

    rng = np.random.default_rng(11)
    kinds = [WorkloadType.PREFILL, WorkloadType.DECODE, WorkloadType.FINETUNE]
    for trial in range(200):
        cfg = SchedulerConfig(tau_task=int(rng.integers(1, 40)), max_decode_batch=int(rng.integers(1, 12)),
                              max_ft_batch=int(rng.integers(1, 4)), tau_mem=float(rng.choice([0.5, 0.9, 1.0])))
        budget = float(rng.choice([50.0, 200.0, 1000.0]))
        hard = budget * float(rng.choice([1.0, 1.5]))
        ests = {}
        queues = (PriorityQueue(PriorityParams(), lambda r: 0.1), FastPriorityQueue(PriorityParams(), lambda r: 0.1),
                  FastPriorityQueue(PriorityParams(), lambda r: 0.1))
        for rid in range(int(rng.integers(0, 60))):
            w = kinds[int(rng.integers(0, 3))]
            pair = PreferencePair(0.5, 4, 4) if w is WorkloadType.FINETUNE else None
            arr = float(rng.integers(0, 5))
            ests[rid] = WorkloadEstimate(mem=float(rng.choice([1.0, 10.0, 60.0, 300.0, rng.random() * 100])),
                                         lat=float(rng.choice([20.0, 120.0, rng.random() * 50])))
            for q in queues:
                q.push(Request(id=rid, tenant=0, workload=w, arrival_time=arr, prompt_tokens=[1], target_output_len=4,
                               pair=pair), 5.0)
        for q in queues:
            q.refresh(5.0)
        est = lambda r: ests[r.id]  # noqa: E731
        a = schedule_iteration(queues[0], budget, cfg, est, 5.0, hard_limit=hard)
        ids = lambda xs: [r.id for r in xs]  # noqa: E731
        for q, native in ((queues[1], True), (queues[2], False)):  # csrc/hostsched.cu and the Python loop
            b = fast_schedule_iteration(q, budget, cfg, est, 5.0, hard_limit=hard, native=native)
            assert ids(a.bin.tasks) == ids(b.bin.tasks), trial
            assert ids(a.requeued) == ids(b.requeued) and ids(a.rejected) == ids(b.rejected)
            assert ids(a.dequeued) == ids(b.dequeued)
            assert (a.bins_opened, a.bins_examined) == (b.bins_opened, b.bins_examined)
            assert (a.bin.used_memory, a.bin.max_latency, a.bin.n_inference, a.bin.n_ft) == \
                (b.bin.used_memory, b.bin.max_latency, b.bin.n_inference, b.bin.n_ft)
            assert [r.priority_state.value for r in a.dequeued] == [r.priority_state.value for r in b.dequeued]
            assert len(queues[0]) == len(q)
        rest = [[q.pop().id for _ in range(len(q))] for q in queues]  # the queues stay in step afterwards
        assert rest[0] == rest[1] == rest[2]


def test_cached_prefix_memo_tracks_trie_changes():
    """GpuPrefixTrie.cached_prefix_len_memo equals a fresh reference walk after every mix of inserts (with
    splits), mark_executed and LRU evictions."""
    import numpy as np

    from paper_2510_03283_b200.kvmanager import GpuPrefixTrie, GroupPool

    rng = np.random.default_rng(5)

    class Tr(GpuPrefixTrie):  # page bookkeeping is not under test here
        def mark_executed(self, leaf, t):
            return super(GpuPrefixTrie, self).mark_executed(leaf, t)

        def lru_offload(self, b, t):
            res = super(GpuPrefixTrie, self).lru_offload(b, t)
            if res.evicted:
                self._epoch += 1
            return res

    tr = Tr(0.1, GroupPool(1))
    prompts, leaves = {}, {}
    base = [rng.integers(0, 4, 24).tolist() for _ in range(4)]
    for step in range(1500):
        op = rng.random()
        if op < 0.35 or not prompts:
            rid = len(prompts)
            p = base[int(rng.integers(0, 4))][: int(rng.integers(1, 24))] + rng.integers(0, 4, int(rng.integers(1, 12))).tolist()
            prompts[rid] = p
            leaves[rid] = tr.insert(p, float(step)).leaf
        elif op < 0.6:
            rid = int(rng.integers(0, len(prompts)))
            if leaves[rid] is not None:
                tr.mark_executed(leaves[rid], float(step))
        elif op < 0.7:
            rid = int(rng.integers(0, len(prompts)))
            if leaves[rid] is not None and all(n.ref_count > 0 for n in leaves[rid].path_nodes()):
                tr.release(leaves[rid])
                leaves[rid] = None
        elif op < 0.75:
            tr.lru_offload(float(rng.integers(1, 20)), float(step))
        for rid in rng.integers(0, len(prompts), 4).tolist():
            assert tr.cached_prefix_len_memo(rid, prompts[rid]) == tr._walk(prompts[rid])[0], (step, rid)


@pytest.mark.parametrize("C,weak", [(160, 0.05), (2000, 1e-4)])
def test_native_head_stats_matches_numpy(C, weak):
    """csrc/hoststats.cu (the product path) equals the numpy restatement bit for bit over many steps:
    first steps (tau unset), full windows, weak heads driving zero-cap repairs, resets, and the uniform split
    -- also at c_total >= 1024, where a packed-digit donor key would lose order."""
    import numpy as np

    from paper_2510_03283_b200.hoststats import BatchedHeadStats

    rng = np.random.default_rng(11)
    H, W, S = 8, 64, 96
    a = BatchedHeadStats(S, H, W, C, 128.0, None)
    b = BatchedHeadStats(S, H, W, C, 128.0, None)
    step_of = np.zeros(S, np.int64)
    for it in range(400):
        n = int(rng.integers(1, 60))
        slots = rng.choice(S, n, replace=False).astype(np.int64)
        reset = slots[rng.random(n) < 0.03]
        if reset.size:
            a.reset(reset)
            b.reset(reset)
            step_of[reset] = 0
        step_of[slots] += 1
        scale = np.where(rng.random((n, H)) < 0.25, weak, 1.0)
        norms = np.maximum(0.0, scale * rng.normal(1.0, 0.1, (n, H)))
        if it % 50 == 7:
            norms[:3] = 0.0  # total <= 0: uniform split
        ka, ra = a.step(slots, step_of[slots], norms)
        kb, rb = b.step_numpy(slots, step_of[slots], norms)
        assert np.array_equal(ka, kb) and np.array_equal(ra, rb)
    for name in ("ring", "count", "pos", "sums", "current", "last_used", "kept"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
    assert np.array_equal(np.isnan(a.tau), np.isnan(b.tau)) and np.array_equal(np.nan_to_num(a.tau), np.nan_to_num(b.tau))


def test_bulk_pair_losses_equal_reference_chain():
    """make_bulk_pair_losses returns exactly env.pair_loss (alignment.py:151-166) while the tenant's mu drifts
    and fine-tune steps move it, for many requests at once."""
    import numpy as np

    from macesim.alignment import AlignmentEnv, TenantParams
    from macesim.workload import PreferencePair, Request, WorkloadType
    from paper_2510_03283_b200.hostfast import make_bulk_pair_losses

    rng = np.random.default_rng(5)
    env = AlignmentEnv.create({0: TenantParams(), 1: TenantParams(mu0=0.7)}, seed=3, beta=1.5)
    reqs = [Request(id=i, tenant=int(rng.integers(0, 2)), workload=WorkloadType.FINETUNE,
                    arrival_time=float(rng.random() * 20), prompt_tokens=[1, 2, 3], target_output_len=4,
                    pair=PreferencePair(float(rng.normal(0.5, 2.0)), 4, 4)) for i in range(300)]
    bulk = make_bulk_pair_losses(env)
    assert bulk is not None
    for it in range(50):
        env.advance_all(float(rng.random() * 0.3))
        if it % 7 == 3:
            env.ft_step(reqs[int(rng.integers(0, len(reqs)))])
        sub = [reqs[int(k)] for k in rng.choice(len(reqs), 40, replace=False)]
        assert bulk(sub) == [env.pair_loss(r) for r in sub]
