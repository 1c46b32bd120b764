"""§8(f)1 measured-cost loop on one B200: calibrate the reference's cost model from the hybrid step, then run
the workload in mode M (tick duration = measured device time).

    python tools/calibrate_b200.py [c4|c3|c2] [--ticks N]

Writes profiles/r2_calib_<wl>.csv (the rows), profiles/r2_profile_<wl>.txt (cost_model.write_profile of the
reference's own calibrate fit) and prints one JSON line: the calibration residuals and a mode-M run of the
workload's trace (TPOT p50/p99 on the measured clock, decode tok/s, evictions / prunes, page budget use)."""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_03283_b200.refpath import ensure_macesim  # noqa: E402

ensure_macesim()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="c4")
    ap.add_argument("--ticks", type=int, default=60)
    args = ap.parse_args()
    from macesim.cost_model import write_profile

    from paper_2510_03283_b200.build import build
    from paper_2510_03283_b200.calibration import calibrated, measure_rows, write_csv
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import WORKLOADS

    build()
    wl = WORKLOADS[args.workload]()
    cfg = wl.model
    w = init_weights(cfg, seed=0, device="cuda")
    model = HybridModel(cfg, wl.train, w, max_slots=1024, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=wl.kv_tokens // 16,
                        decode_pages=1024 * cfg.n_kv_heads * wl.decode_pages_per_head)
    del w
    t0 = time.time()
    rows = measure_rows(model, wl)
    csv = ROOT / "profiles" / f"r2_calib_{wl.name}.csv"
    write_csv(rows, csv)
    rep = calibrated(csv, wl.profile)
    prof_path = ROOT / "profiles" / f"r2_profile_{wl.name}.txt"
    write_profile(rep.profile, prof_path)
    out_dir = ROOT / "gpurun_out"  # the GPU box returns only gpurun_out/
    out_dir.mkdir(exist_ok=True)
    write_csv(rows, out_dir / csv.name)
    write_profile(rep.profile, out_dir / prof_path.name)
    t_cal = time.time() - t0
    # mode M on the workload's own trace: the measured clock decides admissions / bins
    eng = GpuEngine(*wl.engine_args(), model=model, mode="M")
    eng.keep_outputs = False
    eng.time_ticks = True
    done = eng.run_ticks(args.ticks)
    ms = eng.device_ms()
    tbt = eng.measured_tbt_ms()
    ev = [e for e in eng.timeline if e.get("kind") == "cache_event"]
    out = {
        "workload": wl.name, "model": cfg.name, "calibration_rows": len(rows), "calibration_s": round(t_cal, 1),
        "calibrated_profile": {k: getattr(rep.profile, k) for k in ("prefill_lat_per_token", "prefill_mem_per_token",
                                                                 "decode_lat_per_step", "decode_kv_mem_per_token",
                                                                 "ft_lat_per_sample_step", "ft_mem_fixed",
                                                                 "ft_mem_per_token")},
        "residuals": rep.residuals, "points": rep.points_per_workload,
        "mode_m": {"ticks": done, "tokens_per_s": sum(eng.tick_tokens) / (sum(ms) / 1e3),
                   "tick_ms_mean": float(np.mean(ms)), "tpot_ms_p50": float(np.percentile(tbt, 50)) if tbt else None,
                   "tpot_ms_p99": float(np.percentile(tbt, 99)) if tbt else None,
                   "evict_events": sum(1 for e in ev if e["event"] == "evict"),
                   "prune_events": sum(1 for e in ev if e["event"] == "prune"),
                   "page_budget_mb_end": eng.page_budget_mb(), "reference_budget_mb_end": eng._budget()},
    }
    torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
