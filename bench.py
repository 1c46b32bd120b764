#!/usr/bin/env python
"""Hybrid-iteration benchmark (BASELINE.json metric: hybrid-iter tokens/sec/GPU; p50/p99 TPOT; finetune samples/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c3|c2|c1] [--impl ours|reference]

A *step* is one hybrid iteration: one packed bin of Alg. 1 (prefill + decode + DPO fine-tune rows in one
ragged batch) through every decoder layer, plus the masked AdamW update on fine-tune ticks. Default workload
= C4 (BASELINE configs[3]: Llama-3-8B hybrid serving, prefill-heavy trace, one request stream per GPU + NCCL
gradient all-reduce) -- the config the 1/2/4/8-GPU metric is quoted on; one C4 rank fits one B200. Bins are
decided by the UNMODIFIED reference scheduler on its own clock (GpuEngine mode "P": the bins are the
reference's exactly). Tokens per tick = effective (uncached) prefill tokens + decode tokens + fine-tune tokens.

Timed window: ticks [skip + W, skip + W + K) of each rank's trace, with skip chosen from the reference's own
timeline (a cost-model-only run of the unmodified Engine, no execution) so that the window holds fine-tune
ticks at no less than half the trace's steady-state rate -- the window is the hybrid iteration, not a
decode-only stretch. Both arms time exactly these ticks (same ``config``).

Legs (ours):
  e2e    the K ticks through the public API (GpuEngine = the reference Engine.run loop with the override):
         host scheduling, H2D of the tick tables, device work, D2H of every greedy token and fine-tune
         result. Also the measured TPOT: per-request time between tokens on the device clock.
  value  the same K ticks re-issued from a device snapshot with the tick tables pre-packed (inputs
         resident), timed with CUDA events on the launch stream, max over ranks.
  roofline  the dominant kernel class timed per launch with CUDA events over the same ticks: the
         projection GEMMs (tensor-bound) for C4, paged decode attention (HBM-bound) for C1-C3.
  cpu_baseline  rank 0, N=1: the fp32 CPU oracle on a bounded row sample of the same timed ticks, all host
         cores (oracle/sampled.py).
--impl reference: rank 0 only -- the unmodified reference scheduler decides every bin of the same trace, and
  the fp32 CPU oracle executes the same row sample of each timed tick (oracle/sampled.py); same config.
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


def _burst_tflops():
    """The burst cuBLAS bf16 figure (a GEMM timed alone at the boost clock): reported beside the sustained one,
    because the power-capped GEMMs of a long tick can run above cuBLAS's own sustained figure (frac > 1)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["bf16_tflops"])
    return 2250.0


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML, every 2 ms, own thread)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
    }

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self.h = None
        self.error = None
        self._stop = threading.Event()

    def _read(self, h):
        import pynvml

        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        try:
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return sm, r

    def _run(self):
        import pynvml

        try:
            h = self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.error = repr(e)
            return
        while not self._stop.is_set():
            try:
                sm, r = self._read(h)
                self.samples.append((time.perf_counter(), sm, r))
            except Exception as e:  # noqa: BLE001  (one failed poll must not end the sampling)
                self.error = repr(e)
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
        if not smp and self.h is not None:  # the poller recorded nothing: one direct reading right after the window
            try:
                smp = [self._read(self.h)]
            except Exception as e:  # noqa: BLE001
                self.error = repr(e)
        if not smp:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                    "error": self.error}
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
    if model.lora:  # AdamW writes the tenants' adapters and the B columns of the augmented qkv / up weights
        snap["lw"] = {n: t.clone() for n, t in model.lw.items()}
        snap["w"] = {f"layers.{l}.{p}.w": model.w[f"layers.{l}.{p}.w"].clone() for l in model.sel_layers
                     for p in ("qkv", "up")}
        snap["tenant_steps"] = model.tenant_steps.copy()
    else:
        snap["w"] = {n: model.w[n].clone() for n in model.sel}  # AdamW writes only the selected parameters
    snap["adam_step"] = model.adam_step
    snap["kv_mirror"] = model.kv_mirror.state()
    return snap


def restore(model, snap):
    for n, t in snap.items():
        if n in ("w", "lw"):
            for k, v in t.items():
                getattr(model, n)[k].copy_(v)
        elif n == "tenant_steps":
            model.tenant_steps = t.copy()
        elif n == "adam_step":
            model.adam_step = t
        elif n == "kv_mirror":
            model.kv_mirror.restore(t)
        else:
            getattr(model, n).copy_(t)


def make_workload(name, rank, seed=None, lora_tenants=0, lora_rank=16):
    """The workload's trace for this rank: one independent request stream per GPU, seed = base + rank. With
    lora_tenants > 0: that many tenants (the reference's multi-tenant config), each with its own LoRA adapter."""
    from paper_2510_03283_b200.workloads import WORKLOADS, with_tenants

    if name == "c1":
        wl = WORKLOADS["c1"]()
    else:
        base = WORKLOADS[name]().seed if seed is None else seed
        wl = WORKLOADS[name](seed=base + rank)
    if lora_tenants:
        wl = with_tenants(wl, [(0.5 - 0.25 * (u % 5), 0.01 * (1 + u % 3)) for u in range(lora_tenants)], lora_rank)
    return wl


def reference_timeline(wl, n_ticks, capture=None):
    """Run the UNMODIFIED reference Engine on the workload's trace with its own cost-model clock (no model
    execution at all) for n_ticks executed ticks; per tick (n_prefill rows, n_decode, n_ft_pairs). In mode P
    GpuEngine executes exactly these bins (tests/test_engine_c1_gpu.py, tests/test_host_cpu.py)."""
    from macesim.engine import Engine
    from macesim.workload import WorkloadType

    class Probe(Engine):
        def _execute(self, plan):
            t = plan.bin.tasks
            self.comp.append((sum(1 for r in t if r.workload is WorkloadType.PREFILL),
                              sum(1 for r in t if r.workload is WorkloadType.DECODE),
                              sum(1 for r in t if r.workload is WorkloadType.FINETUNE)))
            if capture is not None:
                capture(self, plan)
            super()._execute(plan)
            if len(self.comp) >= n_ticks:
                raise StopIteration

    eng = Probe(*wl.engine_args())
    eng.comp = []
    try:
        eng.run()
    except StopIteration:
        pass
    return eng.comp


def plan_window(wl, steps, warmup, min_skip):
    """skip >= min_skip such that the timed ticks [skip + W, skip + W + K) hold fine-tune ticks at no less than half
    the trace's rate over the scanned steady state (and at least one), from the reference's own timeline."""
    scan = max(4 * steps, 200)
    comp = reference_timeline(wl, min_skip + warmup + steps + scan)
    ft = np.array([c[2] > 0 for c in comp], bool)
    tail = ft[min_skip:]
    rate = float(tail.mean()) if tail.size else 0.0
    need = max(1, int(np.floor(0.5 * rate * steps)))
    for skip in range(min_skip, max(min_skip + 1, len(comp) - warmup - steps + 1)):
        if ft[skip + warmup: skip + warmup + steps].sum() >= need:
            return skip, comp
    return min_skip, comp


def bench_config(wl, args, skip, world):
    """The ``config`` object -- identical in both arms (the driver compares them)."""
    cfg = wl.model
    a, b = skip + args.warmup, skip + args.warmup + args.steps
    return {"workload": f"{wl.name}: {cfg.name} hybrid serving + DPO fine-tune ({wl.name.upper()})",
            "trace": {"arrival_rate": wl.trace_cfg.arrival_rate, "retrain_rate": wl.trace_cfg.retrain_rate,
                      "prompt_len": str(wl.trace_cfg.prompt_len_dist), "output_len": str(wl.trace_cfg.output_len_dist),
                      "seed_rank0": wl.seed, "seeds": "base + rank"},
            "max_decode_batch": wl.sched.max_decode_batch, "max_ft_batch": wl.sched.max_ft_batch,
            "selected_layers": wl.train.n_selected_layers,
            "clock": "reference cost model (mode P: bins identical to the unmodified scheduler)",
            "timed_ticks": [a, b], "warmup_ticks": [skip, a],
            "parallelism": f"request-stream replicas x{world} + NCCL bf16 grad all-reduce",
            "l2": "inputs larger than L2 (weights + KV pages per tick >> 126 MB)",
            **({"lora": {"tenants": wl.n_tenants, "rank": wl.train.lora_rank, "layers": wl.train.n_selected_layers,
                         "trained": "per-tenant adapters only (base frozen)"}} if wl.train.lora_rank else {})}


def run_ours(args, rank, world, lock):
    import torch

    from paper_2510_03283_b200.build import build
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights

    build()
    # MACE_ONE_GPU=1: every rank on cuda:0 (a multi-rank rehearsal of the N>1 path on a one-GPU box, with
    # MACE_DIST_BACKEND=gloo for the gradient all-reduce: NCCL refuses two ranks on one device)
    local = 0 if os.environ.get("MACE_ONE_GPU") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    wl = make_workload(args.workload, rank, args.seed, args.lora_tenants, args.lora_rank)
    cfg = wl.model
    # the timed window from the reference's own timeline (host only); every rank agrees on the largest skip
    min_skip = wl.bench_skip if args.skip is None else args.skip
    skip, comp = plan_window(wl, args.steps, args.warmup, min_skip)
    skip = int(lock.max_over_ranks(float(skip)))
    w = init_weights(cfg, seed=0, device=f"cuda:{local}")
    torch.cuda.synchronize()
    kvtok = args.kv_tokens or wl.kv_tokens
    model = HybridModel(cfg, wl.train, w, device=local, max_slots=args.max_slots, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=kvtok // 16,
                        decode_pages=args.max_slots * cfg.n_kv_heads * wl.decode_pages_per_head,
                        process_group=lock.grad_group if world > 1 else None, n_tenants=wl.n_tenants)
    del w
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", lockstep=lock if world > 1 else None)
    eng.keep_outputs = False
    # ---- ramp the trace to the window (untimed), then warm up
    eng.run_ticks(skip)
    eng.run_ticks(args.warmup)
    torch.cuda.synchronize()
    snap = snapshot(model)
    # ---- e2e: K ticks through the public API (host scheduling + H2D tables + D2H tokens / FT results)
    eng.keep_outputs = True
    eng._dec_out.clear()
    eng.time_ticks = True
    model.tape = []
    h2d0, d2h0 = eng.h2d_bytes, eng.d2h_bytes
    tok0 = len(eng.tick_tokens)
    lock.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    done = eng.run_ticks(args.steps)
    toks_by_req = eng.decoded_tokens()  # D2H of every greedy token of the timed ticks (synchronizes)
    eng._resolve_ref()                  # D2H of the fine-tune pi_ref log-probs
    torch.cuda.synchronize()
    e2e_s = lock.max_over_ranks(time.perf_counter() - t0)
    eng.time_ticks = False
    tbt = eng.measured_tbt_ms()
    tape = model.tape
    model.tape = None
    n_coll = model.tape_collectives(tape)
    if lock.max_over_ranks(float(n_coll)) != lock.min_over_ranks(float(n_coll)):
        raise RuntimeError("ranks recorded different numbers of gradient all-reduces: the replay would deadlock")
    tick_tokens = eng.tick_tokens[tok0:]
    n_tokens = lock.sum_over_ranks(float(sum(tick_tokens)))
    h2d = (eng.h2d_bytes - h2d0) / max(done, 1)
    d2h = (eng.d2h_bytes - d2h0) / max(done, 1)
    # ---- value: replay the same device calls from the snapshot (inputs resident), CUDA events
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
    # ---- roofline of the decode attention (HBM-bound): per-launch CUDA events
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
                 "flops_per_launch_mean": g_flops / max(g_n, 1), "launches": g_n,
                 "peak_burst": _burst_tflops(), "frac_of_burst": g_tflops / _burst_tflops(),
                 "share_note": "per-launch events break the PDL overlap of the value replay: shares are upper bounds"}
    # ---- whole-tick roofline: measured GEMM FLOPs + tensor-core attention FLOPs at the tensor peak,
    # measured decode-attention bytes + row-kernel bytes at the HBM peak, against the device time of the same ticks
    from paper_2510_03283_b200.roofline import tick_extras

    n_sel_l = wl.train.n_selected_layers
    steps_ops = [op for op in tape if op[0] == "step"]
    attn_f = row_b = 0.0
    for op in steps_ops:
        b_ = op[1]
        n_upd = model.n_sel if not model.lora else \
            model.n_sel // model.n_tenants * len({p_.tenant for p_ in b_.ft_pairs})
        e_ = tick_extras(b_, cfg, n_sel_l, n_upd, model.lora)
        attn_f += e_["attn_flops"]
        row_b += e_["row_bytes"]
    roof_ms = 1e3 * ((g_flops + attn_f) / (tc_peak * 1e12) + (sum(byts) + row_b) / (hbm_peak * 1e9))
    dev_ms_rank = ev0.elapsed_time(ev1)
    roof_ms_burst = 1e3 * ((g_flops + attn_f) / (_burst_tflops() * 1e12) + (sum(byts) + row_b) / (hbm_peak * 1e9))
    tick_roof = {"roofline_ms": roof_ms, "measured_ms": dev_ms_rank, "frac": roof_ms / dev_ms_rank if dev_ms_rank else None,
                 "frac_at_burst_tensor_peak": roof_ms_burst / dev_ms_rank if dev_ms_rank else None,
                 "tensor_tflop": (g_flops + attn_f) / 1e12, "gemm_tflop": g_flops / 1e12, "attention_tflop": attn_f / 1e12,
                 "hbm_gb": (sum(byts) + row_b) / 1e9, "decode_attention_gb": sum(byts) / 1e9, "row_kernels_gb": row_b / 1e9,
                 "peaks": {"tensor_tflops": tc_peak, "hbm_gbs": hbm_peak, "source": peak_src},
                 "note": "roofline time = tensor FLOPs / tensor peak + HBM bytes / HBM peak over the timed ticks "
                         "(paper_2510_03283_b200/roofline.py); rank 0's ticks"}
    value = n_tokens / (dev_ms / 1e3)
    e2e = n_tokens / e2e_s
    n_ft_ticks = sum(1 for op in tape if op[0] == "step" and op[1].ft_pairs)
    n_pairs = sum(len(op[1].ft_pairs) for op in tape if op[0] == "step")
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
        "config": bench_config(wl, args, skip, world),
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "roofline": None,
        "clocks": clocks,
        "tpot_ms": {"p50": float(np.percentile(tbt, 50)) if tbt else None,
                    "p99": float(np.percentile(tbt, 99)) if tbt else None, "n": len(tbt),
                    "clock": "measured: device end-of-tick events of the e2e run (reference TBT, engine.py:130-143, "
                             "on the B200 clock; rank 0)"},
        "finetune_samples_per_s": lock.sum_over_ranks(n_pairs) / (dev_ms / 1e3),
        "tick_roofline": tick_roof,
        "ft_ticks_in_timed_region": n_ft_ticks,
        "ft_pairs_in_timed_region": n_pairs,
        "per_gpu_tokens_per_s": value / world,
        "rows_per_tick_mean": float(np.mean(tick_tokens)) if tick_tokens else 0.0,
        "device_ms_per_tick": dev_ms / max(done, 1),
        "host_issue_ms_per_tick": (t_issued - t_on) * 1e3 / max(done, 1),
        "kv_pool_restored_for_replay": "k_pool" in snap,
        "idle_lockstep_rounds": eng.idle_rounds,
    }
    roof_attn = {"bound": "hbm", "kernel": "paged decode attention (attn_decode2_kernel / attn_decode_tc_kernel)",
                 "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                 "peak_source": peak_src, "traffic": None,
                 "share_of_step": attn_ms_total / dev_ms if dev_ms else None,
                 "bytes_per_launch_mean": float(np.mean(byts)) if byts else 0.0,
                 "launches": len(durs)}
    # the roofline line is the workload's dominant kernel class (larger measured share of the step: the projection
    # GEMMs or the paged decode attention); the other one rides along
    dominant_gemm = (roof_gemm["share_of_step"] or 0.0) >= (roof_attn["share_of_step"] or 0.0)
    # dram traffic per launch of each roofline kernel from the committed ncu --set full captures (newest first);
    # a capture is attached only when it profiled this workload's shape (same kernel template)
    cap_gemm, cap_attn = {"c2": (None, "attn_decode"), "c3": (None, "r2s5f_dtc_c3"),
                          "c4": ("gemm_pair", "r2s5f_dtc_c4")}.get(wl.name, (None, None))
    summaries = [ROOT / "profiles" / n for n in ("r2s5f_ncu_full_summary.json", "r2f_ncu_full_summary.json",
                                                  "r2s3_ncu_full_summary.json",
                                                  "r2_ncu_full_summary.json",
                                                  "r1final_ncu_full_summary.json")]
    for cap, target in ((cap_gemm, roof_gemm), (cap_attn, roof_attn)):
        for prof in summaries:
            rows = [r for r in json.loads(prof.read_text()).get(cap, []) if "dram_read" in r] \
                if cap and prof.exists() else []
            if cap and cap.startswith("attn_decode"):
                rows = [r for r in rows if f"<{cfg.head_dim}," in r.get("kernel", "")]
            if rows:
                tr = float(np.mean([r["dram_read"] + r["dram_write"] for r in rows]))
                target["traffic"] = tr
                target["traffic_source"] = f"profiles/{prof.name}[{cap}] ({rows[0]['kernel']}; one ncu --set full capture)"
                if rows[0].get("algorithmic_bytes"):
                    target["traffic_over_algorithmic_in_capture"] = tr / float(np.mean([r["algorithmic_bytes"]
                                                                                          for r in rows]))
                break
    out["roofline"] = roof_gemm if dominant_gemm else roof_attn
    out["roofline_other"] = roof_attn if dominant_gemm else roof_gemm
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, wl, skip, model, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)


def _window_compositions(wl, skip, warmup, steps, max_pos):
    """Row compositions (oracle/sampled.composition) of the reference's warm-up and timed ticks."""
    from oracle.sampled import composition

    comps = []

    def cap(engine, plan):
        if len(engine.comp) > skip:  # engine.comp already holds this tick
            comps.append(composition(engine, plan, max_pos))

    reference_timeline(wl, skip + warmup + steps, capture=cap)
    return comps[:warmup], comps[warmup: warmup + steps]


def cpu_baseline(args, wl, skip, model, budget_s=20.0):
    """fp32 CPU oracle on a bounded row sample of the same timed ticks, all host threads (oracle/sampled.py);
    the weights are the GPU arm's own (bf16 -> fp32 on the host)."""
    import torch

    from oracle.sampled import SampledTickCPU, sample_rows

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    _, timed = _window_compositions(wl, skip, args.warmup, args.steps, wl.model.max_pos)
    # base weights at their model shapes (with per-tenant LoRA the selected layers' device tensors carry the adapter
    # columns [W | B] next to W: the CPU arm runs the base projections, ~0.4% fewer FLOPs than the adapted ones)
    shapes = wl.model.param_shapes()
    w = {}
    for n, t in model.w.items():
        sh = shapes.get(n)
        if sh is not None and t.dim() == 2 and tuple(t.shape) != sh:
            t = t[: sh[0], : sh[1]]
        w[n] = t.float().cpu()
    ex = SampledTickCPU(wl.model, w)
    ex.run(sample_rows(timed[0], min(16, args.cpu_rows)))  # warm (threads, allocator)
    secs = rows = ticks = 0
    for comp in timed:
        rs = sample_rows(comp, args.cpu_rows)
        secs += ex.run(rs)
        rows += len(rs)
        ticks += 1
        if secs > budget_s:
            break
    return {"value": rows / secs if secs else 0.0, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{rows} rows of timed ticks {skip + args.warmup}..{skip + args.warmup + ticks - 1} "
                      f"({args.cpu_rows} per tick, proportional to the tick's prefill / decode / fine-tune rows) "
                      f"through all {wl.model.n_layers} layers of the fp32 oracle, synthetic KV of each row's real "
                      f"context length, no DPO backward (oracle/sampled.py); {secs:.1f} s"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path -- the unmodified macesim scheduler decides every bin, the fp32
    CPU oracle executes a bounded row sample of each timed tick (oracle/sampled.py). Rank 0 only."""
    if rank != 0:
        return
    import torch

    from oracle.sampled import SampledTickCPU, host_weights, sample_rows

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    wl = make_workload(args.workload, 0, args.seed, args.lora_tenants, args.lora_rank)
    min_skip = wl.bench_skip if args.skip is None else args.skip
    skip, _ = plan_window(wl, args.steps, args.warmup, min_skip)
    warm, timed = _window_compositions(wl, skip, args.warmup, args.steps, wl.model.max_pos)
    ex = SampledTickCPU(wl.model, host_weights(wl.model, seed=0, threads=threads))
    for comp in warm[:2]:  # bounded warm-up: threads, allocator, caches
        ex.run(sample_rows(comp, args.cpu_rows))
    secs = rows = 0
    for comp in timed:
        rs = sample_rows(comp, args.cpu_rows)
        secs += ex.run(rs)
        rows += len(rs)
    v = rows / secs if secs else 0.0
    k = len(timed)
    print(json.dumps({
        "impl": "reference", "metric": "hybrid_iter_tokens_per_s", "value": v, "unit": "tokens/s", "n_gpus": world,
        "steps": k, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(k, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(wl, args, skip, world),
        "path": "unmodified macesim Engine bins + fp32 CPU oracle on a row sample of each timed tick (oracle/sampled.py)"
                + ("; base-model rows (the tenants' LoRA adapters, ~1-3% of the FLOPs, are not sampled)"
                   if wl.train.lora_rank else ""),
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"{rows} rows of the {k} timed ticks ({args.cpu_rows} per tick, proportional to the "
                                   f"tick's prefill / decode / fine-tune rows) through all {wl.model.n_layers} layers, "
                                   f"synthetic KV of each row's real context length, no DPO backward; {secs:.1f} s"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=None, help="trace seed of rank 0 (default: the workload's); rank r uses seed + r")
    ap.add_argument("--skip", type=int, default=None, help="minimum ticks before warm-up (default: the workload's)")
    ap.add_argument("--max-slots", type=int, default=1024)
    ap.add_argument("--kv-tokens", type=int, default=None, help="prompt KV capacity in tokens (default: the workload's)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--cpu-rows", type=int, default=128, help="rows of each timed tick the CPU arms execute")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lora-tenants", type=int, default=0, help="per-tenant LoRA adapters: number of tenants (0: off)")
    ap.add_argument("--lora-rank", type=int, default=16)
    args = ap.parse_args()
    from paper_2510_03283_b200.dist import init_from_env

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, lock = init_from_env(os.environ.get("MACE_DIST_BACKEND", "nccl"))
    run_ours(args, rank, world, lock)


if __name__ == "__main__":
    main()
