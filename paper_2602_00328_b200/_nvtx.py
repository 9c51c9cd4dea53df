"""Opt-in NVTX ranges (HARVEST_NVTX=1) around fetch batches, decode steps and
KV operations, for nsys / Nsight timelines ("NVTX ranges per
fetch batch").  No-ops otherwise."""
from __future__ import annotations

import contextlib
import functools
import os

ENABLED = os.environ.get("HARVEST_NVTX", "0") not in ("", "0")


def annotate(name: str):
    """Method decorator: the call runs inside an NVTX range when enabled."""
    def deco(fn):
        if not ENABLED:
            return fn

        @functools.wraps(fn)
        def wrapper(*args, **kwargs):
            with range(name):
                return fn(*args, **kwargs)
        return wrapper
    return deco


@contextlib.contextmanager
def range(name: str):  # noqa: A001 - mirrors torch.cuda.nvtx.range
    if not ENABLED:
        yield
        return
    import torch
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()
