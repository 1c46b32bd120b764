"""Decode-window compaction (mace_kv_compact) on the B200. C1's trace with long decodes (96 tokens) and a larger
per-request KV capacity (CacheConfig c_total 1200): the reference's allocate_capacity (cache.py:318-352) gives the
weak heads windows of ~9 slots and its prune trim (engine.py:496-529) slides them every tick, so they often
straddle a page boundary they do not need. With compaction after every trim, such windows are re-based: their K/V
rows move down inside their pages and the emptied pages return to the free stack. Checked: the device allocator
equals the host mirror (free-stack top, every dec_base), pages were reclaimed, and every tick still matches the
fp32 oracle, whose decode windows are semantic (tests/parity_util.py) -- attention reads exactly the moved rows."""
import dataclasses

import pytest
import torch

from parity_util import check_records

pytestmark = pytest.mark.gpu


def _engine(record=True):
    from macesim.distributions import parse_dist
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    wl = dataclasses.replace(wl, trace_cfg=dataclasses.replace(
        wl.trace_cfg, duration=2.0, output_len_dist=parse_dist("constant:value=96")),
        cache=dataclasses.replace(wl.cache, c_total=1200))
    w = init_weights(wl.model, seed=0)
    model = HybridModel(wl.model, wl.train, w, max_slots=128, max_prompt_len=wl.max_prompt_len, prompt_groups=1024)
    return GpuEngine(*wl.engine_args(), model=model, mode="P", record=record), model, w, wl


def _allocator_agrees(model):
    top, status = model.kv_status()
    assert status == 0 and top == model.kv_mirror.free
    base = model.dec_base.cpu().numpy()
    assert (base == model.kv_mirror.base[: base.shape[0]]).all()
    return base


def test_compaction_after_trims_keeps_parity(ctx):
    eng, model, w, wl = _engine()
    model.compact_max_window = 16
    eng.run_ticks(60)
    torch.cuda.synchronize()
    base = _allocator_agrees(model)
    assert (base % 16 != 0).any(), "no window was re-based"
    assert model.compaction_pages > 0 and model.compaction_bytes > 0
    st = check_records(eng, w, wl.model, wl.train, label="C1 long decodes + compaction after trims")
    assert st["tokens"] > 500


def test_on_demand_compaction_reclaims_pages(ctx):
    eng, model, w, wl = _engine()
    eng.run_ticks(30)
    torch.cuda.synchronize()
    free0 = model.kv_mirror.free
    got = model.compact_windows()  # what step() runs when a tick's page pops exceed the free pages
    torch.cuda.synchronize()
    assert got > 0 and model.kv_mirror.free == free0 + got
    _allocator_agrees(model)
    eng.run_ticks(20)
    torch.cuda.synchronize()
    _allocator_agrees(model)
    st = check_records(eng, w, wl.model, wl.train, label="C1 long decodes + one on-demand compaction")
    assert st["tokens"] > 300
