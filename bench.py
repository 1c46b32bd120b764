#!/usr/bin/env python
"""Hybrid-iteration benchmark (BASELINE.json metric: hybrid-iter tokens/sec/GPU; p50/p99 TPOT; finetune samples/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c1] [--impl ours|reference]

A *step* is one hybrid iteration (one packed bin of Alg. 1: prefill + decode + DPO fine-tune rows in
one ragged batch, through every decoder layer, plus the masked AdamW update on fine-tune ticks).
Default workload = BASELINE configs[1] (GPT-2 small hybrid serving + DPO, 1 B200, Poisson trace), bins
decided by the UNMODIFIED reference scheduler on its own clock (GpuEngine mode "P", so the bins are the
reference's exactly). Tokens counted per tick = effective (uncached) prefill tokens + decode tokens +
fine-tune tokens processed.

Legs (ours):
  e2e    K ticks through the public API (GpuEngine, i.e. the reference Engine.run loop with the
         override): host scheduling, H2D of the tick tables, device work, D2H of every greedy token.
  value  the same K ticks re-issued from a device snapshot with the tick tables pre-packed
         (inputs resident), timed with CUDA events on the launch stream, max over ranks.
  roofline  the dominant kernel (paged decode attention) timed per launch with CUDA events over the
         same ticks; achieved = algorithmic K/V+Q+O bytes / duration vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  rank 0, N=1: the fp32 CPU oracle executing the reference scheduler's bins on all host
         cores for a bounded sample (oracle/ref_arm.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def _peaks():
    """(HBM GB/s, dense bf16 TF/s, source). The tensor peak is the SUSTAINED cuBLAS figure: the GEMMs run
    inside a long step (B200_PROFILING.md: burst for a kernel timed alone, sustained inside a long step)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML, every 2 ms, own thread)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
    }

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        import pynvml

        h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self._stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            try:
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.samples.append((time.perf_counter(), sm, r))
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t is not None:
            self.t.join()

    def summary(self, t0: float | None = None, t1: float | None = None):
        """Samples inside the timed window [t0, t1] (host perf_counter); all samples if no window."""
        smp = [(s, r) for t, s, r in self.samples if (t0 is None or t >= t0) and (t1 is None or t <= t1)]
        if not smp:  # window shorter than one NVML poll: take the nearest samples around it
            smp = [(s, r) for t, s, r in self.samples][-3:]
        if not smp:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for _, r in smp for bit, n in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in smp), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(smp)}


def snapshot(model):
    """Device state the timed ticks mutate. The KV pools are restored only when a copy fits next to them:
    without it the replay re-writes the same pages with the same (deterministic) values, and only pages that
    the original run evicted and re-used read other (finite) KV content -- same bytes, same launches."""
    import torch

    names = ["ptab", "dtab", "dec_base", "dec_first", "dec_end", "free_stack", "free_top", "last_token", "master",
             "m", "v"]
    pool_bytes = 2 * model.k_pool.numel() * model.k_pool.element_size()
    if pool_bytes < 0.6 * torch.cuda.mem_get_info(model.dev)[0]:
        names = ["k_pool", "v_pool"] + names
    snap = {n: getattr(model, n).clone() for n in names}
    snap["w"] = {n: model.w[n].clone() for n in model.sel}  # AdamW writes only the selected parameters
    snap["adam_step"] = model.adam_step
    return snap


def restore(model, snap):
    for n, t in snap.items():
        if n == "w":
            for k, v in t.items():
                model.w[k].copy_(v)
        elif n == "adam_step":
            model.adam_step = t
        else:
            getattr(model, n).copy_(t)


def make_workload(args, rank):
    """The workload's trace for this rank: one independent request stream per GPU, seed = base + rank."""
    from paper_2510_03283_b200.workloads import WORKLOADS

    if args.workload == "c1":
        return WORKLOADS["c1"]()
    base = WORKLOADS[args.workload]().seed if args.seed is None else args.seed
    return WORKLOADS[args.workload](seed=base + rank)


def run_ours(args, rank, world, lock):
    import torch

    from paper_2510_03283_b200 import ops
    from paper_2510_03283_b200.build import build
    from paper_2510_03283_b200.config import TrainConfig
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import WORKLOADS

    build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    wl = make_workload(args, rank)
    cfg = wl.model
    w = init_weights(cfg, seed=0, device=f"cuda:{local}")
    torch.cuda.synchronize()
    kvtok = args.kv_tokens or wl.kv_tokens
    model = HybridModel(cfg, wl.train, w, device=local, max_slots=args.max_slots, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=kvtok // 16,
                        decode_pages=args.max_slots * cfg.n_kv_heads * wl.decode_pages_per_head,
                        process_group=lock.grad_group if world > 1 else None)
    del w
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", lockstep=lock if world > 1 else None)
    eng.keep_outputs = False
    # ---- ramp the trace to steady state (untimed), then warm up
    args.skip = wl.bench_skip if args.skip is None else args.skip
    eng.run_ticks(args.skip)
    eng.run_ticks(args.warmup)
    torch.cuda.synchronize()
    snap = snapshot(model)
    # ---- e2e: K ticks through the public API (host scheduling + H2D tables + D2H tokens)
    eng.keep_outputs = True
    eng._dec_out.clear()
    model.tape = []
    h2d0, d2h0 = eng.h2d_bytes, eng.d2h_bytes
    tok0 = len(eng.tick_tokens)
    lock.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    done = eng.run_ticks(args.steps)
    toks_by_req = eng.decoded_tokens()  # D2H of every greedy token of the timed ticks (synchronizes)
    torch.cuda.synchronize()
    e2e_s = lock.max_over_ranks(time.perf_counter() - t0)
    tape = model.tape
    model.tape = None
    tick_tokens = eng.tick_tokens[tok0:]
    n_tokens = lock.sum_over_ranks(float(sum(tick_tokens)))
    h2d = (eng.h2d_bytes - h2d0) / max(done, 1)
    d2h = (eng.d2h_bytes - d2h0) / max(done, 1)
    # ---- value: replay the same device calls from the snapshot (inputs resident), CUDA events
    launches0 = model.ctx.launches
    clk = ClockSampler(local).__enter__()  # sampling runs through the warm replay and the timed region
    restore(model, snap)
    model.replay(tape)  # warm replay
    restore(model, snap)
    torch.cuda.synchronize()
    lock.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_on = time.perf_counter()
    ev0.record()
    l0 = model.ctx.launches
    model.replay(tape)
    ev1.record()
    t_issued = time.perf_counter()
    ev1.synchronize()
    t_off = time.perf_counter()
    launches = model.ctx.launches - l0
    time.sleep(0.01)
    clk.__exit__()
    dev_ms = lock.max_over_ranks(ev0.elapsed_time(ev1))
    clocks = clk.summary(t_on, t_off)
    # ---- roofline of the dominant kernel: paged decode attention, per-launch CUDA events
    restore(model, snap)
    hbm_peak, tc_peak, peak_src = _peaks()
    model.instrument = []
    model.replay(tape)
    torch.cuda.synchronize()
    durs, byts = [], []
    for ev_a, ev_b, nbytes in model.instrument:
        durs.append(ev_a.elapsed_time(ev_b))
        byts.append(nbytes)
    model.instrument = None
    attn_ms_total = sum(durs)
    achieved = (sum(byts) / (attn_ms_total / 1e3)) / 1e9 if durs else 0.0
    # ---- roofline of the GEMMs (tensor-bound): CUDA events around every GEMM launch of the same ticks
    restore(model, snap)
    model.gemm_instrument = []
    model.replay(tape)
    torch.cuda.synchronize()
    g_ms = sum(x[0] for x in model.gemm_instrument)
    g_flops = sum(x[1] for x in model.gemm_instrument)
    g_n = sum(x[2] for x in model.gemm_instrument)
    model.gemm_instrument = None
    g_tflops = g_flops / (g_ms / 1e3) / 1e12 if g_ms else 0.0
    roof_gemm = {"bound": "tensor", "kernel": "gemm_tc_kernel / gemm_tc2_kernel (all projections, fwd + FT bwd)",
                 "achieved": g_tflops, "peak": tc_peak, "unit": "TFLOP/s", "frac": g_tflops / tc_peak if tc_peak else None,
                 "peak_source": peak_src, "traffic": None, "share_of_step": g_ms / dev_ms if dev_ms else None,
                 "flops_per_launch_mean": g_flops / max(g_n, 1), "launches": g_n}
    one_tick_ms = dev_ms / max(done, 1)
    value = n_tokens / (dev_ms / 1e3)
    e2e = n_tokens / e2e_s
    # TPOT proxies: per-tick device time of the timed ticks (decode tokens emitted once per tick)
    lat = eng.metrics.latency_summary()
    out = {
        "metric": "hybrid_iter_tokens_per_s",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": done,
        "warmup": args.warmup,
        "ms_per_step": dev_ms / max(done, 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (reference generate_trace Poisson trace; seeded random-init weights at the real shapes)",
        "config": {"workload": f"{wl.name}: {cfg.name} hybrid serving + DPO ({args.workload})", "model": cfg.name,
                   "arrival_rate": wl.trace_cfg.arrival_rate, "retrain_rate": wl.trace_cfg.retrain_rate,
                   "max_decode_batch": wl.sched.max_decode_batch, "selected_layers": wl.train.n_selected_layers,
                   "clock": "reference cost model (mode P: bins identical to the unmodified scheduler)",
                   "skip_ticks": args.skip, "parallelism": f"request-stream replicas x{world} + NCCL grad all-reduce",
                   "l2": "inputs larger than L2 (weights + KV pages per tick >> 126 MB)",
                   "kv_pool_restored_for_replay": "k_pool" in snap,
                   "per_gpu_tokens_per_s": value / world,
                   "rows_per_tick_mean": float(np.mean(tick_tokens)) if tick_tokens else 0.0},
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "roofline": None,
        "clocks": clocks,
        "tpot_reference_clock_ms": {"p50": lat["tbt_p50"], "p99": lat["tbt_p99"]},
        "device_ms_per_tick": one_tick_ms,
        "host_issue_ms_per_tick": (t_issued - t_on) * 1e3 / max(done, 1),
        "finetune_samples_per_s": None,
    }
    roof_attn = {"bound": "hbm", "kernel": "attn_decode_kernel (paged decode attention)",
                 "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                 "peak_source": peak_src, "traffic": None,
                 "share_of_step": attn_ms_total / dev_ms if dev_ms else None,
                 "bytes_per_launch_mean": float(np.mean(byts)) if byts else 0.0,
                 "launches": len(durs)}
    # the roofline line is the workload's dominant single kernel: decode attention for the decode-carrying
    # C1-C3 ticks (the largest single kernel of the step; the GEMM line aggregates ~60 launches of several GEMM
    # shapes), the projection GEMMs for the prefill-heavy C4; the other one rides along
    dominant_gemm = wl.name == "c4"
    # DRAM traffic per launch of the same kernel from the committed ncu --set full capture of this workload
    # (tools/ncu_capture.sh -> profiles/r1final_ncu_full_summary.json; cold-cache, serialised)
    cap = {"c2": "attn_decode", "c3": "attn_decode_tc", "c4": "gemm_pair"}.get(wl.name)
    prof = ROOT / "profiles" / "r1final_ncu_full_summary.json"
    if cap and prof.exists():
        rows = [r for r in json.loads(prof.read_text()).get(cap, []) if "dram_read" in r]
        if rows:
            tr = float(np.mean([r["dram_read"] + r["dram_write"] for r in rows]))
            target = roof_gemm if dominant_gemm else roof_attn
            target["traffic"] = tr
            target["traffic_source"] = f"profiles/r1final_ncu_full_summary.json[{cap}] ({rows[0]['kernel']})"
            if rows[0].get("algorithmic_bytes"):
                target["traffic_over_algorithmic_in_capture"] = tr / float(np.mean([r["algorithmic_bytes"] for r in rows]))
    out["roofline"] = roof_gemm if dominant_gemm else roof_attn
    out["roofline_other"] = roof_attn if dominant_gemm else roof_gemm
    n_ft_ticks = sum(1 for op in tape if op[0] == "step" and op[1].ft_pairs)
    n_pairs = sum(len(op[1].ft_pairs) for op in tape if op[0] == "step")
    out["finetune_samples_per_s"] = lock.sum_over_ranks(n_pairs) / (dev_ms / 1e3)
    out["config"]["ft_ticks_in_timed_region"] = n_ft_ticks
    if args.workload == "c4" and not args.no_cpu_baseline:
        # the fp32 CPU oracle of Llama-3-8B needs 32 GB of host weights and ~200 s per prefill-heavy tick
        out["cpu_baseline"] = {"unavailable": "c4 (Llama-3-8B): one fp32 CPU oracle tick exceeds the bounded "
                                              "sample; the c2 line carries the CPU baseline"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, wl, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out))


def cpu_baseline(args, wl, budget_s=20.0):
    """fp32 CPU oracle on the reference scheduler's bins, all host threads, bounded sample."""
    import torch

    from oracle.ref_arm import make_reference_engine_cls
    from paper_2510_03283_b200.config import selected_param_names
    from paper_2510_03283_b200.weights import init_weights

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    Eng = make_reference_engine_cls()
    cfg = wl.model
    w = init_weights(cfg, seed=0)
    eng = Eng(*wl.engine_args())
    eng.setup(cfg, w, wl.train, selected_param_names(cfg, wl.train), wl.seed)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        before = eng._done
        eng.run_ticks(1)
        if eng._done == before:
            break
    secs = sum(eng.tick_secs)
    toks = sum(eng.tick_tokens)
    return {"value": toks / secs if secs else 0.0, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"first {eng._done} ticks of the {wl.name} trace (reference bins from tick 0, incl. ramp-up), "
                      f"{toks} tokens in {secs:.1f} s of oracle compute"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (unmodified macesim scheduler + fp32 oracle math)."""
    if rank != 0:
        return
    import torch

    from oracle.ref_arm import make_reference_engine_cls
    from paper_2510_03283_b200.config import selected_param_names
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import WORKLOADS

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    wl = make_workload(args, 0)
    cfg = wl.model
    Eng = make_reference_engine_cls()
    eng = Eng(*wl.engine_args())
    eng.setup(cfg, init_weights(cfg, seed=0), wl.train, selected_param_names(cfg, wl.train), wl.seed)
    # bounded sample: the fp32 CPU path needs ~10-80 s for one early (prefill / fine-tune heavy) C2 tick, so the
    # warm-up is one tick (tick 0: oracle caches and threads warm) and the timed ticks stop at a wall-clock
    # budget; the same ticks-from-0 sample as the cpu_baseline leg of the GPU arm (the whole arm ends in minutes)
    t_w = time.perf_counter()
    while eng._done < min(args.warmup, 1) and time.perf_counter() - t_w < args.ref_seconds / 6:
        before = eng._done
        eng.run_ticks(1)
        if eng._done == before:
            break
    n0 = len(eng.tick_tokens)
    t0 = time.perf_counter()
    while len(eng.tick_tokens) - n0 < args.steps and time.perf_counter() - t0 < args.ref_seconds:
        before = eng._done
        eng.run_ticks(1)
        if eng._done == before:
            break
    wall = time.perf_counter() - t0
    toks = sum(eng.tick_tokens[n0:])
    k = len(eng.tick_tokens) - n0
    v = toks / wall if wall else 0.0
    print(json.dumps({
        "impl": "reference", "metric": "hybrid_iter_tokens_per_s", "value": v, "unit": "tokens/s", "n_gpus": world,
        "steps": k, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(k, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{wl.name}: {cfg.name} hybrid serving + DPO ({args.workload})", "model": cfg.name,
                   "path": "unmodified macesim Engine bins + fp32 CPU oracle arithmetic (oracle/ref_arm.py)"},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"ticks {n0}..{n0 + k} of the trace (from tick 0; warm-up and timed ticks "
                                   f"bounded by {args.ref_seconds:.0f} s of wall clock), {toks} tokens"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=None, help="trace seed of rank 0 (default: the workload's); rank r uses seed + r")
    ap.add_argument("--skip", type=int, default=None, help="ticks to reach steady state before warm-up (default: the workload's)")
    ap.add_argument("--max-slots", type=int, default=1024)
    ap.add_argument("--kv-tokens", type=int, default=None, help="prompt KV capacity in tokens (default: the workload's)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=120.0, help="--impl reference: wall-clock bound of the timed ticks")
    args = ap.parse_args()
    from paper_2510_03283_b200.dist import init_from_env

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, lock = init_from_env("nccl")
    run_ours(args, rank, world, lock)


if __name__ == "__main__":
    main()
