"""Trace v2 (pair content): round trip, the reference's v1 files still read, reader errors name the line, and
GpuEngine feeds a ContentPair's own responses into the fine-tune rows (truncated to the model's positions)."""
import json

import pytest

from fakes import FakeModel


def _trace():
    from paper_2510_03283_b200.workloads import c1

    return c1().trace()


def test_v2_round_trip_and_v1_compat(tmp_path):
    from macesim.workload import write_trace
    from paper_2510_03283_b200.engine import synthetic_pair_tokens
    from paper_2510_03283_b200.tracev2 import ContentPair, read_trace_any, read_trace_v2, write_trace_v2

    tr = _trace()
    content = lambda r: synthetic_pair_tokens(0, r.id, r.pair.tokens_chosen, r.pair.tokens_rejected + 3, 50000)  # noqa: E731
    p2 = tmp_path / "t.v2"
    write_trace_v2(tr, p2, content=content)
    back = read_trace_v2(p2)
    assert len(back) == len(tr)
    for a, b in zip(tr, back):
        assert (a.id, a.tenant, a.workload, a.arrival_time, a.prompt_tokens, a.target_output_len) == \
               (b.id, b.tenant, b.workload, b.arrival_time, b.prompt_tokens, b.target_output_len)
        if a.pair is not None:
            c, r = content(a)
            assert isinstance(b.pair, ContentPair) and b.pair.chosen == c and b.pair.rejected == r
            assert b.pair.initial_margin == a.pair.initial_margin
            assert (b.pair.tokens_chosen, b.pair.tokens_rejected) == (len(c), len(r))
    p3 = tmp_path / "t.v2b"
    write_trace_v2(back, p3)  # ContentPairs need no content callback
    assert p3.read_text() == p2.read_text()
    p1 = tmp_path / "t.v1"
    write_trace(_trace(), p1)
    v1 = read_trace_any(p1)
    assert [r.id for r in v1] == [r.id for r in tr]


def test_v2_reader_errors(tmp_path):
    from macesim.workload import TraceParseError
    from paper_2510_03283_b200.tracev2 import read_trace_v2

    p = tmp_path / "bad"
    p.write_text("mace-trace-v2\n0\t0\tfinetune\t0.1\t1,2\t4\t0.5\t\t\n")
    with pytest.raises(TraceParseError, match="line 2"):
        read_trace_v2(p)
    p.write_text("mace-trace-v1\n")
    with pytest.raises(TraceParseError, match="line 1"):
        read_trace_v2(p)


def test_engine_uses_pair_content(tmp_path):
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.tracev2 import ContentPair, from_jsonl
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    recs = [{"prompt": list(range(5, 5 + 40 + i)), "chosen": [7 + i] * (9 + i), "rejected": [11 + i] * (4 + 2 * i)}
            for i in range(6)]
    jl = tmp_path / "pairs.jsonl"
    jl.write_text("\n".join(json.dumps(r) for r in recs) + "\n")
    trace = sorted(wl.trace() + from_jsonl(jl, arrival_rate=20.0, seed=1, first_id=10_000), key=lambda r: r.arrival_time)
    args = list(wl.engine_args())
    args[0] = trace
    fm = FakeModel(wl.model, wl.train, max_prompt_len=wl.max_prompt_len)
    eng = GpuEngine(*args, model=fm, mode="P")
    eng.keep_outputs = False
    eng.run()
    seen = {}
    for c in fm.calls:
        if c[0] == "step":
            for p in c[1].ft_pairs:
                seen[p.rid] = (p.chosen, p.rejected)
    for i, r in enumerate(recs):
        rid = 10_000 + i
        assert rid in seen, "every content pair ran at least one fine-tune step"
        assert seen[rid] == (r["chosen"], r["rejected"])
    assert isinstance(next(t for t in trace if t.id == 10_000).pair, ContentPair)
