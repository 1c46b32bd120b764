"""Trace format v2: fine-tune requests carry their preference pair's token content.

The reference's ``mace-trace-v1`` (workload.py:221-283) stores, per request, 7 tab-separated fields -- id,
tenant, workload, arrival, prompt token ids, target output length, initial margin -- so a preference pair is
only its LENGTHS (tokens_chosen = tokens_rejected = target_output_len, workload.py:205,265). A real DPO step
needs the chosen / rejected responses themselves. ``mace-trace-v2`` appends two fields:

    8  chosen response token ids  (comma-separated; empty for prefill requests)
    9  rejected response token ids (comma-separated; empty for prefill requests)

and the pair lengths become the content lengths (chosen and rejected may differ). Everything else -- field
order, number formatting (repr floats), the workload names, the error classes and their "line N:" messages --
follows the reference's reader / writer, so a v1 file still reads through ``read_trace_any`` (content then
comes from the builder-defined synthetic stream, engine.synthetic_pair_tokens).

``ContentPair`` is the reference's PreferencePair plus the content; GpuEngine.build_batch uses the content when
present. ``from_jsonl`` ingests pre-tokenized preference data ({"prompt": [...], "chosen": [...],
"rejected": [...]} per line, e.g. HH-RLHF / SHP after offline tokenization) into fine-tune requests.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

from .refpath import ensure_macesim

ensure_macesim()
from macesim.workload import (  # noqa: E402
    TRACE_SCHEMA,
    PreferencePair,
    Request,
    TraceParseError,
    WorkloadType,
    read_trace,
)

TRACE_SCHEMA_V2 = "mace-trace-v2"


@dataclass
class ContentPair(PreferencePair):
    chosen: list[int] = field(default_factory=list)
    rejected: list[int] = field(default_factory=list)

    @classmethod
    def of(cls, initial_margin: float, chosen: list[int], rejected: list[int]) -> "ContentPair":
        return cls(initial_margin, len(chosen), len(rejected), list(chosen), list(rejected))


def _ids(xs) -> str:
    return ",".join(str(int(t)) for t in xs)


def write_trace_v2(trace: list[Request], path: str | Path, content=None) -> None:
    """v1's records (workload.py:221-240 field formatting) + chosen / rejected ids. ``content(req)`` supplies the
    pair content of requests whose pair is not a ContentPair (e.g. engine.synthetic_pair_tokens)."""
    lines = [TRACE_SCHEMA_V2]
    for req in trace:
        margin = "" if req.pair is None else repr(req.pair.initial_margin)
        ch = rj = ""
        if req.pair is not None:
            if isinstance(req.pair, ContentPair):
                c, r = req.pair.chosen, req.pair.rejected
            elif content is not None:
                c, r = content(req)
            else:
                raise ValueError(f"request {req.id}: pair without content (pass content=...)")
            ch, rj = _ids(c), _ids(r)
        lines.append("\t".join((str(req.id), str(req.tenant), req.workload.value, repr(req.arrival_time),
                                _ids(req.prompt_tokens), str(req.target_output_len), margin, ch, rj)))
    Path(path).write_text("\n".join(lines) + "\n")


def read_trace_v2(path: str | Path) -> list[Request]:
    lines = Path(path).read_text().splitlines()
    if not lines or lines[0].strip() != TRACE_SCHEMA_V2:
        raise TraceParseError(f"line 1: expected header {TRACE_SCHEMA_V2!r}")
    trace: list[Request] = []
    for lineno, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        parts = line.split("\t")
        if len(parts) != 9:
            raise TraceParseError(f"line {lineno}: expected 9 fields, got {len(parts)}")
        try:
            workload = WorkloadType(parts[2])
            ids = lambda s: [int(t) for t in s.split(",")] if s else []  # noqa: E731
            pair = None
            if workload is WorkloadType.FINETUNE:
                if parts[6] == "":
                    raise ValueError("missing initial_margin for finetune request")
                c, r = ids(parts[7]), ids(parts[8])
                if not c or not r:
                    raise ValueError("finetune request without chosen / rejected content")
                pair = ContentPair.of(float(parts[6]), c, r)
            elif parts[6] != "" or parts[7] != "" or parts[8] != "":
                raise ValueError("initial_margin / pair content must be empty for non-finetune request")
            trace.append(Request(id=int(parts[0]), tenant=int(parts[1]), workload=workload,
                                 arrival_time=float(parts[3]), prompt_tokens=ids(parts[4]),
                                 target_output_len=int(parts[5]), pair=pair))
        except TraceParseError:
            raise
        except (ValueError, KeyError) as exc:
            raise TraceParseError(f"line {lineno}: {exc}") from exc
    return trace


def read_trace_any(path: str | Path) -> list[Request]:
    """v2 (with pair content) or the reference's v1 (lengths only)."""
    head = Path(path).read_text().split("\n", 1)[0].strip()
    if head == TRACE_SCHEMA_V2:
        return read_trace_v2(path)
    if head == TRACE_SCHEMA:
        return read_trace(path)
    raise TraceParseError(f"line 1: expected header {TRACE_SCHEMA_V2!r} or {TRACE_SCHEMA!r}")


def from_jsonl(path: str | Path, arrival_rate: float, seed: int = 0, tenant: int = 0, first_id: int = 0,
               initial_margin: float = 0.0) -> list[Request]:
    """Fine-tune requests from pre-tokenized preference records, Poisson arrivals at ``arrival_rate``."""
    import numpy as np

    rng = np.random.default_rng([seed, 409])
    t = 0.0
    out = []
    for i, line in enumerate(Path(path).read_text().splitlines()):
        if not line.strip():
            continue
        rec = json.loads(line)
        t += float(rng.exponential(1.0 / arrival_rate))
        c, r = list(rec["chosen"]), list(rec["rejected"])
        out.append(Request(id=first_id + len(out), tenant=tenant, workload=WorkloadType.FINETUNE, arrival_time=t,
                           prompt_tokens=list(rec["prompt"]), target_output_len=max(len(c), len(r)),
                           pair=ContentPair.of(float(rec.get("margin", initial_margin)), c, r)))
    return out
