"""Decode-attention microbenchmark (B200): B decode rows, each over a prompt of n_pv tokens plus a short decode
window per KV head, in the head-major paged pools; CUDA-event timing of mace_attn_fwd (decode items only, warm,
inputs larger than L2), algorithmic bytes = every visible K and V row once + q / o rows.
    python tools/decode_bench.py [impl hd Hq Hkv B n_pv] ...   (impl 1: CUDA-core streaming, 2: tcgen05 swap-AB)"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx, MaceKvLayout  # noqa: E402
from paper_2510_03283_b200.build import build  # noqa: E402

PG = 16
CASES = [(2, 128, 32, 8, 256, 1500), (2, 64, 32, 8, 256, 1920), (1, 64, 12, 12, 200, 400), (2, 128, 32, 8, 64, 2000)]


def run(ctx, impl, hd, Hq, Hkv, B, n_pv, dec=24, iters=20, seed=0):
    rng = np.random.default_rng(seed)
    dev = "cuda"
    W = (Hq + 2 * Hkv) * hd
    npg = (n_pv + PG - 1) // PG
    maxpp, maxdp = npg + 1, (dec + PG - 1) // PG + 1
    n_groups = B * npg
    n_head_pages = n_groups * Hkv + B * Hkv * maxdp + 8
    ptab = np.zeros((B, maxpp), np.int32)
    ptab[:, :npg] = rng.permutation(n_groups).reshape(B, npg)
    dtab = (n_groups * Hkv + np.arange(B * Hkv * maxdp, dtype=np.int32)).reshape(B, Hkv, maxdp)
    dec_base = np.zeros((B, Hkv), np.int32)
    dec_first = np.zeros((B, Hkv), np.int32)
    dec_end = np.full(B, dec, np.int32)
    seqs = [[1, i, 1, i, n_pv, 0, 0, 0] for i in range(B)]
    nch = max(1, -(-npg // 128))
    items = [[i, h, (c << 16) | nch, (i * Hkv + h) * nch] for i in range(B) for h in range(Hkv) for c in range(nch)]
    items.sort(key=lambda it: -1)
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    d = dict(ptab=t(ptab), dtab=t(dtab), dec_base=t(dec_base), dec_first=t(dec_first), dec_end=t(dec_end))
    qkv = torch.randn(B, W, device=dev).bfloat16()
    kp = torch.randn(n_head_pages, PG, hd, device=dev).bfloat16()
    vp = torch.randn(n_head_pages, PG, hd, device=dev).bfloat16()
    seq_t = torch.tensor(seqs, dtype=torch.int32, device=dev)
    items_t = torch.tensor(items, dtype=torch.int32, device=dev)
    ws = torch.empty(len(items) * (2 * (Hq // Hkv) + (Hq // Hkv) * hd), device=dev)
    cnt = torch.zeros(B * Hkv, dtype=torch.int32, device=dev)
    work = torch.zeros(1, dtype=torch.int64, device=dev)
    lay = MaceKvLayout(ptab=d["ptab"].data_ptr(), max_prompt_pages=maxpp, dtab=d["dtab"].data_ptr(),
                       max_dec_pages=maxdp, dec_base=d["dec_base"].data_ptr(), dec_first=d["dec_first"].data_ptr(),
                       dec_end=d["dec_end"].data_ptr(), free_stack=None, free_top=None, stack_cap=0, n_kv_heads=Hkv)
    out = torch.zeros(B, Hq * hd, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def call():
        ops.attn_fwd(ctx, qkv, Hq, Hkv, hd, seq_t, None, items_t, lay, kp, vp, out, dec_workspace=ws, dec_counters=cnt,
                     dec_work=work, decode_impl=impl)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        flush.zero_()  # > L2: every launch reads its K / V from HBM
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    byts = B * Hkv * (n_pv + dec) * hd * 2 * 2 + B * Hq * hd * 2 * 2
    return {"impl": impl, "hd": hd, "Hq": Hq, "Hkv": Hkv, "B": B, "n_pv": n_pv, "us": ms * 1e3,
            "GBps": byts / (ms / 1e3) / 1e9, "bytes": byts}


def main():
    build()
    ctx = Ctx(0)
    argv = sys.argv[1:]
    cases = [tuple(int(x) for x in argv[i: i + 6]) for i in range(0, len(argv), 6)] if len(argv) >= 6 else CASES
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    for c in cases:
        r = run(ctx, *c)
        r["frac"] = r["GBps"] / peak
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
