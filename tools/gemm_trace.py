"""Phase timeline of the tcgen05 GEMM from inside the kernel (%globaltimer per CTA; trace build).

    python tools/gemm_trace.py M N K mode
Builds libmace_b200_trace.so (-DMACE_GEMM_TRACE) and prints, over CTAs, the median / max offset (us)
from the earliest CTA entry of: entry, setup done, PDL wait done, first TMA issued, first stage full,
each tile's last MMA issued, epilogue start / end, exit."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["MACE_LIB"] = "libmace_b200_trace.so"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_03283_b200.build import build  # noqa: E402

build(variant="trace", defines=("MACE_GEMM_TRACE",))
from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx  # noqa: E402

M, N, K, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
dbg = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # 1: MMA-rate probe, 2: TMA-rate probe
ctx = Ctx(0)
ws = torch.empty(64 << 20, device="cuda")
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(N, K, device="cuda").bfloat16()
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode.startswith("f32") else torch.bfloat16)
tr = torch.zeros(1024 * 64, dtype=torch.int64, device="cuda")
import time  # noqa: E402
t_end = time.time() + 1.0  # warm the clocks: ~1 s of back-to-back launches
while time.time() < t_end:
    for _ in range(50):
        ops.gemm(ctx, a, b, out, mode=mode, workspace=ws)
    torch.cuda.synchronize()
torch.cuda.synchronize()
ctx.L.mace_debug_gemm_trace.argtypes = [__import__("ctypes").c_void_p, __import__("ctypes").c_int]
ctx.L.mace_debug_gemm_trace(tr.data_ptr(), dbg)
ops.gemm(ctx, a, b, out, mode=mode, workspace=ws)
torch.cuda.synchronize()
t_all = tr.view(1024, 64).cpu().numpy()
used = t_all[:, 0] > 0
t = t_all[used, :32].astype(np.float64)
cyc = t_all[used, 32:].astype(np.float64)
ok = (cyc[:, 4] > 0) & (cyc[:, 9] > 0)
if ok.any():
    mm = cyc[ok, 9] - cyc[ok, 4]
    print(f"first_full -> t0_epi_start (MMAs complete): median {np.median(mm):.0f} cycles")
ok = (cyc[:, 4] > 0) & (cyc[:, 8] > 0)
if ok.any():
    mm = cyc[ok, 8] - cyc[ok, 4]
    print(f"mainloop first_full -> t0_mma_done: median {np.median(mm):.0f} cycles "
          f"({np.median(mm) / max(1, (K + 63) // 64):.0f} cycles per k-block of the first tile's split)")
t0 = t[:, 0].min()
names = {0: "entry", 1: "setup", 2: "pdl_wait", 3: "first_tma", 4: "first_full", 31: "exit"}
for i in range(5):
    names[8 + 4 * i] = f"t{i}_mma_done"
    names[9 + 4 * i] = f"t{i}_epi_start"
    names[10 + 4 * i] = f"t{i}_epi_end"
print(f"{used.sum()} CTAs")
for k in sorted(names):
    col = t[:, k]
    v = col[col > 0]
    if v.size:
        print(f"{names[k]:14s} n={v.size:4d} min {1e-3 * (v.min() - t0):7.2f} med {1e-3 * (np.median(v) - t0):7.2f} "
              f"max {1e-3 * (v.max() - t0):7.2f} us")
