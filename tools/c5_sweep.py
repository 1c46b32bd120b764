"""C5: Llama-3-8B KV-memory-pressure sweep on the C4 trace, one B200.

For each capacity (MB) the unmodified reference scheduler (mode P clock) drives the B200 hybrid step for a
fixed tick window; the reference's fine-tune memory charge is set from the device: ft_mem_per_token =
HybridModel.ft_bytes_per_token() (the FT-row buffers the step really allocates), ft_mem_fixed = 0 (the
selected-parameter optimizer state is resident, outside the budget). Reported per capacity: reference
cache events (evict / prune, engine.py:364-372,520-529), rejections, KV pages freed on the device (trie
evictions, prune trims and the decode-window compactions with the bytes they moved), TPOT p50/p99 (reference
clock), device tokens/s over the window. The smallest capacities leave the reference's budget below the trie's
residency, so its LRU offload (cache.py:217-238) evicts page groups on the device.
    python tools/c5_sweep.py [--ticks 64] [--caps 20480,24576,32768,40960,81920,184320]
"""
import argparse
import gc
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200.build import build  # noqa: E402
from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.kvmanager import KvCapacityError  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.weights import init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import c4  # noqa: E402
from macesim.distributions import parse_dist  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ticks", type=int, default=96)
ap.add_argument("--caps", default="20480,24576,32768,40960,81920,184320")
ap.add_argument("--pool-gb", type=float, default=112.0, help="prompt KV pool the B200 holds next to the 8B model")
ap.add_argument("--output-mean", type=float, default=4.0,
                help="geometric mean output length (C4: 32). The reference evicts only when the QUEUE HEAD does not fit "
                     "(engine.py:375-389, every tick before planning): decode rows (priority 3) head the queue while any "
                     "request decodes and their prefix nodes stay referenced, so short outputs are what let finished "
                     "prefixes pile up in the trie and a prefill head trigger the LRU offload")
args = ap.parse_args()
build()
caps = [float(x) for x in args.caps.split(",")]
wl0 = c4()
cfg = wl0.model
w = init_weights(cfg, seed=0, device="cuda")
kv_tok_bytes = cfg.kv_bytes_per_token()
pool_tokens = int(args.pool_gb * 1e9 / kv_tok_bytes) // 16 * 16
rows = []
for cap in caps:
    wl = c4(capacity_mb=cap)
    wl = replace(wl, trace_cfg=replace(wl.trace_cfg, output_len_dist=parse_dist(f"geometric:mean={args.output_mean}")))
    model = HybridModel(cfg, wl.train, w, device=0, max_slots=1024, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps,
                        prompt_groups=min(wl.kv_tokens, pool_tokens) // 16,
                        decode_pages=1024 * cfg.n_kv_heads * wl.decode_pages_per_head)
    ft_mb = model.ft_bytes_per_token() / 2**20
    prof = replace(wl.profile, ft_mem_fixed=0.0, ft_mem_per_token=ft_mb)
    args_e = list(wl.engine_args())
    args_e[1] = prof
    eng = GpuEngine(*args_e, model=model, mode="P")
    eng.keep_outputs = False
    eng.time_ticks = True
    freed0 = eng.pool.in_use
    t0 = time.perf_counter()
    err = None
    try:
        done = eng.run_ticks(args.ticks)
    except KvCapacityError as e:  # the reference's budget asks for more KV than one B200 holds
        done, err = eng.ticks_done, str(e)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev_ms = sum(a.elapsed_time(b) for a, b in eng.tick_device_ms)
    ev = [e for e in eng.timeline if e.get("kind") == "cache_event"]
    lat = eng.metrics.latency_summary()
    row = {
        "capacity_mb": cap, "output_len_mean": args.output_mean, "ft_mem_per_token_mb": ft_mb, "ticks": done,
        "evict_events": sum(1 for e in ev if e.get("event") == "evict"),
        "evicted_nodes": sum(e.get("nodes", 0) for e in ev if e.get("event") == "evict"),
        "evicted_mb": -sum(e.get("bytes_mb", 0.0) for e in ev if e.get("event") == "evict"),
        "prune_events": sum(1 for e in ev if e.get("event") == "prune"),
        "pruned_slots": sum(e.get("slots", 0) for e in ev if e.get("event") == "prune"),
        "rejected": len(eng.metrics.rejected_ids),
        "prompt_groups_in_use": eng.pool.in_use, "prompt_groups_capacity": eng.pool.n,
        "tokens": int(sum(eng.tick_tokens)), "device_ms": dev_ms,
        "device_tokens_per_s": sum(eng.tick_tokens) / (dev_ms / 1e3) if dev_ms else None,
        "e2e_tokens_per_s": sum(eng.tick_tokens) / wall,
        "tpot_p50_ms": lat["tbt_p50"], "tpot_p99_ms": lat["tbt_p99"], "error": err,
        "kv_compaction_heads": model.compaction_pages, "kv_compaction_bytes": model.compaction_bytes,
        "kv_compacted_tokens": model.kv_mirror.compacted_tokens,
        "decode_pages_free": model.kv_mirror.free, "decode_pages": model.kv_mirror.n_pages,
        "trie_groups_released_by_evict": getattr(eng.trie, "groups_released_by_evict", None),
    }
    rows.append(row)
    print(json.dumps(row), flush=True)
    del eng, model
    gc.collect()  # the engine holds reference cycles (norm stream, trie); free the device pools now
    torch.cuda.empty_cache()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/c5_sweep.json").write_text(json.dumps(rows, indent=1))
