"""Host-side logic on CPU (no GPU): the drop-in keeps the reference's decisions bit-identical, and the
KV page manager's tables always resolve to the right KV rows (incl. prefix sharing, splits,
copy-on-diverge and LRU eviction)."""
import json
from pathlib import Path

import pytest

from fakes import FakeModel

GOLD = Path(__file__).parent / "golden" / "c1_reference.json"


def _engine(wl, **kw):
    from paper_2510_03283_b200.engine import GpuEngine

    fm = FakeModel(wl.model, wl.train, max_prompt_len=wl.max_prompt_len, **kw)
    eng = GpuEngine(*wl.engine_args(), model=fm, mode="P")
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


@pytest.mark.parametrize("policy", ["HybridNoPrefix", "HybridNoPrune", "Periodic", "Sync", "HybridNoBin"])
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
    """The batched head-stats/prune bookkeeping (hoststats.py) reproduces the reference's per-row
    _exec_decode exactly: same timeline (prune events carry MB deltas), kept[] and metrics."""
    from paper_2510_03283_b200.workloads import WORKLOADS

    def run(fast):
        wl = WORKLOADS[wl_name]()
        eng, fm = _engine(wl, prompt_groups=1 << 15, max_slots=1024)
        eng.fast_host = fast
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
    for H, C in ((8, 160), (12, 160), (4, 10), (3, 7)):
        hs = BatchedHeadStats(1, H, 4, C, 128, None)
        means = rng.random((4000, H)) * rng.choice([1.0, 0.01], size=(4000, H))
        means[rng.random((4000, H)) < 0.1] = 0.0
        means[:5] = 0.0
        got = hs._allocate(means)
        want = np.array([allocate_capacity(m.tolist(), C) for m in means])
        assert (got == want).all()
