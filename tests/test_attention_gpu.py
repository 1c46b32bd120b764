"""Ragged paged attention (tcgen05 prefill/FT tiles + streamed decode rows) vs a torch fp32 reference."""
import math

import numpy as np
import pytest
import torch

from paper_2510_03283_b200 import ops
from paper_2510_03283_b200._lib import MaceKvLayout

pytestmark = pytest.mark.gpu
PG = 16


def _build(hd, Hq, Hkv, seed, prefill=((200, 120), (40, 40), (300, 1)),
           decode=((150, 37), (16, 1), (33, 100), (1537, 60)), ft=(130, 77, 256)):
    g = torch.Generator().manual_seed(seed)
    rng = np.random.default_rng(seed)
    dev = "cuda"
    W = (Hq + 2 * Hkv) * hd
    n_slots = len(prefill) + len(decode)
    maxpp = 128
    maxdp = 16
    # page allocation: prompt groups then per-head decode pages
    total_groups = sum((n + PG - 1) // PG for n, _ in prefill) + sum((n + PG - 1) // PG for n, _ in decode)
    dec_pages_needed = len(decode) * Hkv * maxdp
    n_head_pages = total_groups * Hkv + dec_pages_needed + 8
    groups = rng.permutation(total_groups)
    ptab = np.zeros((n_slots, maxpp), np.int32)
    dtab = np.zeros((n_slots, Hkv, maxdp), np.int32)
    dec_base = np.zeros((n_slots, Hkv), np.int32)
    dec_first = np.zeros((n_slots, Hkv), np.int32)
    dec_end = np.zeros((n_slots,), np.int32)
    gi = 0
    seqs, tc_items, dec_items = [], [], []
    row = 0
    slot = 0
    # prefill sequences
    for n_pv, q_len in prefill:
        npg = (n_pv + PG - 1) // PG
        ptab[slot, :npg] = groups[gi: gi + npg]
        gi += npg
        seqs.append([0, row, q_len, slot, n_pv, n_pv, -1, 0])
        row += q_len
        slot += 1
    # decode sequences: random per-head windows
    free_dec = list(range(total_groups * Hkv, n_head_pages))
    rng.shuffle(free_dec)
    for n_pv, de in decode:
        npg = (n_pv + PG - 1) // PG
        ptab[slot, :npg] = groups[gi: gi + npg]
        gi += npg
        dec_end[slot] = de
        for h in range(Hkv):
            db = 16 * int(rng.integers(0, max(1, (de - 1) // 16 + 1)))
            df = int(rng.integers(db, de))  # window [df, de) non-empty
            dec_base[slot, h] = db
            dec_first[slot, h] = df
            for r in range((de - 1 - db) // 16 + 1):
                dtab[slot, h, r] = free_dec.pop()
        seqs.append([1, row, 1, slot, n_pv - 1, 0, len(dec_items), 0])
        row += 1
        slot += 1
    for n in ft:
        seqs.append([2, row, n, -1, 0, n, -1, 0])
        row += n
    T = row
    for si, s in enumerate(seqs):
        if s[0] == 1:
            nch = max(1, -(-((s[4] + 15) // 16) // 32))
            for h in range(Hkv):
                base = len(dec_items)
                for ch in range(nch):
                    dec_items.append([si, h, (ch << 16) | nch, base])
        else:
            for hq in range(Hq):
                for qb in range((s[2] + 127) // 128):
                    tc_items.append([si, hq, qb, 0])
    qkv = (torch.randn(T, W, generator=g)).bfloat16()
    kp = torch.randn(n_head_pages, PG, hd, generator=g).bfloat16()
    vp = torch.randn(n_head_pages, PG, hd, generator=g).bfloat16()
    host = dict(qkv=qkv, kp=kp, vp=vp, ptab=ptab, dtab=dtab, dec_base=dec_base, dec_first=dec_first,
                dec_end=dec_end, seqs=seqs)
    d = {k: (torch.from_numpy(v).to(dev) if isinstance(v, np.ndarray) else v.to(dev)) for k, v in host.items() if k != "seqs"}
    d["seqs"] = torch.tensor(seqs, dtype=torch.int32, device=dev)
    d["tc_items"] = torch.tensor(tc_items, dtype=torch.int32, device=dev).reshape(-1, 4) if tc_items else None
    d["dec_items"] = torch.tensor(dec_items, dtype=torch.int32, device=dev).reshape(-1, 4) if dec_items else None
    d["dec_ws"] = torch.empty(len(dec_items) * (2 * (Hq // Hkv) + (Hq // Hkv) * hd), device=dev)
    d["dec_cnt"] = torch.zeros(n_slots * Hkv, dtype=torch.int32, device=dev)
    d["dec_work"] = torch.zeros(1, dtype=torch.int64, device=dev)
    rng.shuffle(dec_items)  # any order: items carry their partial slot
    lay = MaceKvLayout(ptab=d["ptab"].data_ptr(), max_prompt_pages=maxpp, dtab=d["dtab"].data_ptr(), max_dec_pages=maxdp,
                       dec_base=d["dec_base"].data_ptr(), dec_first=d["dec_first"].data_ptr(),
                       dec_end=d["dec_end"].data_ptr(), free_stack=None, free_top=None, stack_cap=0, n_kv_heads=Hkv)
    return host, d, lay, T


def _reference(host, Hq, Hkv, hd, T, lse=None):
    qkv = host["qkv"].float()
    kp, vp = host["kp"].float(), host["vp"].float()
    G = Hq // Hkv
    out = torch.zeros(T, Hq, hd)
    for s in host["seqs"]:
        kind, q0, ql, slot, n_pv, kv_len = s[:6]
        q = qkv[q0: q0 + ql, : Hq * hd].reshape(ql, Hq, hd)
        for hq in range(Hq):
            h = hq // G
            if kind == 2:
                K = qkv[q0: q0 + ql, (Hq + h) * hd: (Hq + h + 1) * hd]
                V = qkv[q0: q0 + ql, (Hq + Hkv + h) * hd: (Hq + Hkv + h + 1) * hd]
            else:
                toks = [(host["ptab"][slot, t // PG] * Hkv + h, t % PG) for t in range(n_pv)]
                if kind == 1:
                    db, df, de = host["dec_base"][slot, h], host["dec_first"][slot, h], host["dec_end"][slot]
                    toks += [(host["dtab"][slot, h, (j - db) // PG], j % PG) for j in range(df, de)]
                K = torch.stack([kp[p, r] for p, r in toks])
                V = torch.stack([vp[p, r] for p, r in toks])
            m = K.shape[0]
            sc = q[:, hq] @ K.t() / math.sqrt(hd)
            if kind != 1:
                qlog = torch.arange(ql)[:, None] + (m - ql)
                sc = sc.masked_fill(torch.arange(m)[None, :] > qlog, float("-inf"))
            if kind == 2 and s[7] > 0:  # preference-pair key hole (MaceSeq hole0 / hole_len)
                h0, h1 = s[6], s[6] + s[7]
                keys, rows = torch.arange(m)[None, :], torch.arange(ql)[:, None]
                sc = sc.masked_fill((rows >= h1) & (keys >= h0) & (keys < h1), float("-inf"))
            out[q0: q0 + ql, hq] = torch.softmax(sc, -1) @ V
            if lse is not None:
                lse[q0: q0 + ql, hq] = torch.logsumexp(sc, -1)
    return out


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("hd,Hq,Hkv", [(32, 8, 8), (64, 12, 12), (64, 32, 8), (128, 8, 2), (128, 32, 8)])
def test_attention_ragged(ctx, hd, Hq, Hkv, impl):
    host, d, lay, T = _build(hd, Hq, Hkv, seed=hd + Hq)
    out = torch.zeros(T, Hq * hd, dtype=torch.bfloat16, device="cuda")
    hn = torch.zeros(T, Hq, device="cuda")
    lse = torch.zeros(T, Hq, device="cuda")
    for _ in range(2):  # twice: the chunk-merge counters must come back zeroed
        ops.attn_fwd(ctx, d["qkv"], Hq, Hkv, hd, d["seqs"], d["tc_items"], d["dec_items"], lay, d["kp"], d["vp"], out,
                     lse=lse, head_norm=hn, dec_workspace=d["dec_ws"], dec_counters=d["dec_cnt"],
                     dec_work=d["dec_work"], decode_impl=impl)
    assert int(d["dec_cnt"].abs().sum()) == 0
    if impl == 1:  # the ticket counter is back at zero, so a fresh buffer at a reused address is safe
        assert int(d["dec_work"].abs().sum()) == 0
    torch.cuda.synchronize()
    ref = _reference(host, Hq, Hkv, hd, T)
    got = out.float().cpu().reshape(T, Hq, hd)
    err = (got - ref).abs().max().item()
    assert err < 3e-2, f"max abs err {err}"
    # decode rows: head norms are ||o|| of the fp32 output
    for s in host["seqs"]:
        if s[0] == 1:
            r = s[1]
            want = ref[r].norm(dim=-1)
            assert torch.allclose(hn[r].cpu(), want, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("hd,Hq,Hkv", [(64, 12, 12), (64, 32, 8), (128, 32, 8)])
def test_attention_tc_pairs_and_pair_hole(ctx, hd, Hq, Hkv, pairs):
    """The tensor-core prefill / FT path with single 128-row query blocks and with query-block PAIRS (two tiles per
    CTA, csrc/attention_fa2.cu), on ragged prefill + FT sequences, one FT sequence laid out as a preference pair
    with a key hole: outputs and LSE against the fp32 reference."""
    host, d, lay, T = _build(hd, Hq, Hkv, seed=7 * hd + Hq, decode=(), ft=(130, 77, 300, 520))
    for s in host["seqs"]:
        if s[0] == 2 and s[2] == 300:
            s[6], s[7] = 120, 61  # rows >= 181 do not see keys [120, 181)
    seqs = torch.tensor(host["seqs"], dtype=torch.int32, device="cuda")
    blk = 256 if pairs else 128
    items = [[si, hq, qb, 0] for si, s in enumerate(host["seqs"]) if s[0] != 1 for hq in range(Hq)
             for qb in range((s[2] + blk - 1) // blk)]
    items_t = torch.tensor(items, dtype=torch.int32, device="cuda")
    out = torch.zeros(T, Hq * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros(T, Hq, device="cuda")
    ops.attn_fwd(ctx, d["qkv"], Hq, Hkv, hd, seqs, items_t, None, lay, d["kp"], d["vp"], out, lse=lse,
                 tc_pairs=pairs)
    torch.cuda.synchronize()
    lse_ref = torch.zeros(T, Hq)
    ref = _reference(host, Hq, Hkv, hd, T, lse=lse_ref)
    got = out.float().cpu().reshape(T, Hq, hd)
    err = (got - ref).abs().max().item()
    assert err < 3e-2, f"max abs err {err}"
    assert (lse.cpu() - lse_ref).abs().max().item() < 2e-2
