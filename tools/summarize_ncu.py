"""Summarise the ncu captures of tools/ncu_capture.sh into profiles/ (run in the build container)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

OUT = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles")
TAG = sys.argv[2] if len(sys.argv) > 2 else "r1"
SRC = Path("gpurun_out")
M = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active": "uniform_pipe_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__cycles_active.avg": "cycles",
}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, name in M.items():
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[i]
                if name in ("dram_read", "dram_write") and isinstance(v, float):
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if name == "duration_us" and isinstance(v, float):
                    v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
                d[name] = v
        out.append(d)
    return out


def main():
    OUT.mkdir(exist_ok=True)
    summary = {}
    for name in ("attn_decode", "gemm", "attn_fa", "attn_decode_tc", "gemm_pair", "attn_fa_c4", "attn_bwd_c4", "adamw",
                 "paging"):
        rep = SRC / f"{name}.ncu-rep"
        if rep.exists():
            summary[name] = raw(rep)
    # algorithmic bytes per decode-attention launch of the C2 replay (the launch-list run: same snapshot, so its
    # first ticks are the ones the --set full capture replays; later profile_tick runs overwrite the plain file)
    src = SRC / "decode_attn_bytes_launchlist.json"
    if not src.exists():
        src = SRC / "decode_attn_bytes.json"
    algo = json.loads(src.read_text()) if src.exists() else []
    if "attn_decode" in summary and algo:
        for j, d in enumerate(summary["attn_decode"]):
            a = algo[12 + j]  # ncu -s 12: launches 13.. of the 2-tick replay
            d["algorithmic_bytes"] = a
            d["traffic_bytes"] = d["dram_read"] + d["dram_write"]
            d["traffic_over_algorithmic"] = d["traffic_bytes"] / a
    (OUT / f"{TAG}_ncu_full_summary.json").write_text(json.dumps(summary, indent=1))
    lines = [f"# {TAG} ncu --set full captures (C2 / C3 / C4 steady state, tools/ncu_capture.sh; cold-cache, serialised)", ""]
    for name, rows in summary.items():
        lines.append(f"## {name}")
        for d in rows:
            lines.append("- " + ", ".join(f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}" for k, v in d.items()))
        lines.append("")
    (OUT / f"{TAG}_ncu_full_summary.md").write_text("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
