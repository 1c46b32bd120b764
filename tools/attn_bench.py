"""Time the tensor-core prefill / fine-tune attention on dense causal sequences (CUDA events, warm).
    python tools/attn_bench.py [hd Hq Hkv n_seqs seq_len] ...   (MACE_ATTN_OLD=1: the first tc kernel)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx, MaceKvLayout  # noqa: E402
from paper_2510_03283_b200.build import build  # noqa: E402

build()
ctx = Ctx(0)
BWD = "--bwd" in sys.argv
PAIRS = "--pairs" in sys.argv  # query-block pairs: two 128-row tiles per CTA (csrc/attention_fa2.cu)
ATOMIC = "--atomic" in sys.argv  # backward dQ by fp32 atomics instead of the ordered (deterministic) accumulation
argv = [a for a in sys.argv[1:] if a not in ("--bwd", "--pairs", "--atomic")]
cases = [(128, 32, 8, 16, 1280), (128, 32, 8, 4, 2048), (64, 12, 12, 16, 512), (64, 32, 8, 16, 1920)]
if len(argv) >= 5:
    cases = [tuple(int(x) for x in argv[:5])]
for hd, Hq, Hkv, S, n in cases:
    W = (Hq + 2 * Hkv) * hd
    T = S * n
    qkv = torch.randn(T, W, device="cuda").bfloat16()
    seqs = torch.tensor([[2, i * n, n, -1, 0, n, -1, 0] for i in range(S)], dtype=torch.int32, device="cuda")
    items = []
    blk = 256 if PAIRS else 128
    nb = (n + blk - 1) // blk
    for si in range(S):
        for hq in range(Hq):
            for qb in range(nb):
                items.append([si, hq, qb, (min(qb * blk + blk, n) + 127) // 128])
    items.sort(key=lambda x: -x[3])
    items = torch.tensor(items, dtype=torch.int32, device="cuda")
    out = torch.empty(T, Hq * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(T, Hq, device="cuda")
    lay = MaceKvLayout(ptab=None, max_prompt_pages=0, dtab=None, max_dec_pages=0, dec_base=None, dec_first=None,
                       dec_end=None, free_stack=None, free_top=None, stack_cap=0, n_kv_heads=Hkv)

    def run():
        ops.attn_fwd(ctx, qkv, Hq, Hkv, hd, seqs, items, None, lay, None, None, out, lse=lse, tc_pairs=PAIRS)

    if BWD:  # time the backward of the same sequences (forward once for o / lse)
        run()
        dout = torch.randn(T, Hq * hd, device="cuda").bfloat16()
        kblk = 128 if hd >= 64 else 64
        nkb = (n + kblk - 1) // kblk
        bitems = sorted([[si, h, kb, nkb - kb] for si in range(S) for h in range(Hkv) for kb in range(nkb)],
                        key=lambda x: -x[3])
        bitems = torch.tensor(bitems, dtype=torch.int32, device="cuda")
        dqkv = torch.zeros(T, W, device="cuda")

        def run():  # noqa: F811
            dqkv.zero_()
            ops.attn_bwd(ctx, qkv, out, dout, lse, Hq, Hkv, hd, seqs, bitems, dqkv=dqkv, ordered=not ATOMIC)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    flops = S * (10 if BWD else 4) * Hq * hd * (n * (n + 1) / 2)
    print(f"hd={hd} Hq={Hq} Hkv={Hkv} seqs={S}x{n}: {us:9.1f} us  {flops / us / 1e6:7.1f} TF/s  (items {items.shape[0]})")
