"""Locate the unmodified reference package ``macesim`` (the host scheduler this path plugs into).

The reference is never copied into this repo. Search order:
  1. $MACE_REF_PATH (a directory containing the ``macesim`` package)
  2. <repo>/baseline/_ref  (pip --target install of /root/reference/pkg; git-ignored, travels with
     the snapshot to the GPU box)
  3. /root/reference/pkg/src (the read-only mount, present only in the build container)
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

_REPO = Path(__file__).resolve().parents[1]


def candidates() -> list[Path]:
    out = []
    env = os.environ.get("MACE_REF_PATH")
    if env:
        out.append(Path(env))
    out += [_REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")]
    return out


def ensure_macesim() -> Path:
    for c in candidates():
        if (c / "macesim" / "engine.py").exists():
            if str(c) not in sys.path:
                sys.path.append(str(c))
            return c
    raise ImportError(
        "macesim (the reference scheduler/engine) not found; install it with\n"
        "  python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>"
    )
