"""The CPU arms' tick sample (oracle/sampled.py, bench.py's cpu_baseline leg and --impl reference): the bin
compositions the unmodified reference hands to Engine._execute, in the GPU path's row layout (one sequence per
preference pair), the proportional row sample and its execution through the fp32 oracle -- on C1, so a broken
sample path fails here and not at round end."""
import bench
from oracle.sampled import KIND_DECODE, KIND_FT, KIND_PREFILL, SampledTickCPU, host_weights, sample_rows


def test_window_compositions_match_the_gpu_row_layout():
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    warm, timed = bench._window_compositions(wl, 0, 2, 10, wl.model.max_pos)
    comps = warm + timed
    assert len(comps) == 12
    kinds = {r[0] for c in comps for r in c["rows"]}
    assert {KIND_PREFILL, KIND_DECODE, KIND_FT} <= kinds
    for c in comps:
        n = {k: sum(1 for r in c["rows"] if r[0] == k) for k in (KIND_PREFILL, KIND_DECODE, KIND_FT)}
        assert n[KIND_PREFILL] == c["n_prefill"] and n[KIND_DECODE] == c["n_decode"] and n[KIND_FT] == c["n_ft"]
        # per pair: prompt + chosen + the re-entered last prompt token + rejected; predicting rows = n_c + n_r
        ft = [r for r in c["rows"] if r[0] == KIND_FT]
        assert sum(r[3] for r in ft) <= len(ft)


def test_sampled_rows_run_through_the_oracle():
    from paper_2510_03283_b200.config import ModelConfig
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    _, timed = bench._window_compositions(wl, 0, 1, 3, wl.model.max_pos)
    cfg = ModelConfig("tiny-2l", "llama", 2, 128, 4, 4, 32, 256, 50000, max_pos=4096)
    ex = SampledTickCPU(cfg, host_weights(cfg, seed=0, threads=2))
    for comp in timed:
        rows = sample_rows(comp, 16)
        assert 0 < len(rows) <= 16 + 3  # proportional, at least one row per present kind
        assert ex.run(rows) > 0
