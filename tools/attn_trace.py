"""Per-tile timeline of the warp-specialised attention kernel (CTA 0, clock64; trace build).
    python tools/attn_trace.py [hd Hq Hkv n_seqs seq_len]"""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["MACE_LIB"] = "libmace_b200_atrace.so"
import torch  # noqa: E402

from paper_2510_03283_b200.build import build  # noqa: E402

build(variant="atrace", defines=("MACE_ATTN_TRACE",))
from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx, MaceKvLayout  # noqa: E402

hd, Hq, Hkv, S, n = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (128, 32, 8, 4, 2048)
ctx = Ctx(0)
W = (Hq + 2 * Hkv) * hd
qkv = torch.randn(S * n, W, device="cuda").bfloat16()
seqs = torch.tensor([[2, i * n, n, -1, 0, n, -1, 0] for i in range(S)], dtype=torch.int32, device="cuda")
nb = (n + 127) // 128
items = sorted([[si, hq, qb, qb + 1] for si in range(S) for hq in range(Hq) for qb in range(nb)], key=lambda x: -x[3])
items = torch.tensor(items, dtype=torch.int32, device="cuda")
out = torch.empty(S * n, Hq * hd, dtype=torch.bfloat16, device="cuda")
lay = MaceKvLayout(ptab=None, max_prompt_pages=0, dtab=None, max_dec_pages=0, dec_base=None, dec_first=None,
                   dec_end=None, free_stack=None, free_top=None, stack_cap=0, n_kv_heads=Hkv)
for _ in range(20):
    ops.attn_fwd(ctx, qkv, Hq, Hkv, hd, seqs, items, None, lay, None, None, out)
tr = torch.zeros(3 * 8 * 64, dtype=torch.int64, device="cuda")
ctx.L.mace_debug_attn_trace.argtypes = [ctypes.c_void_p]
ctx.L.mace_debug_attn_trace(tr.data_ptr())
ops.attn_fwd(ctx, qkv, Hq, Hkv, hd, seqs, items, None, lay, None, None, out)
torch.cuda.synchronize()
t = tr.view(3, 8, 64).cpu().numpy()
t0 = t[t > 0].min()
names = ["s_ready", "S_loaded", "xchg", "exp_done", "o_done", "p_arrive"]
print("tile | WG0: " + " ".join(f"{x:>9s}" for x in names) + " | MMA: issue_S issue_PV")
for g in range(24):
    w0 = " ".join(f"{(t[0, e, g] - t0) if t[0, e, g] else -1:9d}" for e in range(6))
    print(f"{g:4d} | {w0} | {t[2, 0, g] - t0 if t[2,0,g] else -1:9d} {t[2, 1, g] - t0 if t[2,1,g] else -1:9d}")
print("WG1 exp_done - s_ready per tile:", [int(t[1, 3, g] - t[1, 0, g]) for g in range(1, 16)])
print("WG0 period:", [int(t[0, 0, g + 1] - t[0, 0, g]) for g in range(0, 16)])
