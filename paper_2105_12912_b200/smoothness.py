"""Workflow selection (mirrors P/smoothness.py:26-37, 111-136).

The 1.09-bit rule: a stream expected to Huffman-code at or below
RLE_THRESHOLD_BITS bits/symbol goes to RLE + VLE.  Exact mode uses the true
average code length of the device-built code book (K2 returns sum(c*len) and
the total; the division is done here exactly as numpy does it).  Estimate
mode evaluates the entropy + redundancy bracket on the cap-bin histogram --
host arithmetic on a few KB, kept on the host so the floats are bit-identical
with numpy (the entropy bounds are host-side by design).

``analyze`` / ``sample_madogram`` (P/smoothness.py:40-108, 139-188) are
profiling tools outside the compress path; not built.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .errors import DataError

RLE_THRESHOLD_BITS = 1.09


class Workflow(IntEnum):
    """Symbol-stream codec recorded in archives (P/smoothness.py:32-37)."""

    HUFFMAN = 0
    RLE = 1
    RLE_VLE = 2


@dataclass(frozen=True)
class WorkflowDecision:
    chosen: Workflow
    b_estimate: float
    basis: str  # "exact" | "bounds"
    threshold: float = RLE_THRESHOLD_BITS


def estimate_bits(counts: np.ndarray) -> float:
    """Midpoint of [H + R-, H + R+] (P/codebook.py:81-87, P/smoothness.py:127-130)."""
    from .codebook import entropy_report

    rep = entropy_report(np.asarray(counts, np.int64))
    return (rep.b_lo + rep.b_hi) / 2.0


def select_workflow(counts, mode: str = "exact", threshold: float = RLE_THRESHOLD_BITS,
                    override: Workflow | None = None) -> WorkflowDecision:
    """P/smoothness.py:111-136; exact mode builds the code book on the GPU (K2)."""
    from .codebook import Codebook

    counts = np.asarray(counts, np.int64)
    if mode == "exact":
        book = Codebook.from_counts(counts)
        b = book.average_bits(counts)
        basis = "exact"
    elif mode == "estimate":
        b = estimate_bits(counts)
        basis = "bounds"
    else:
        raise DataError(f"unknown selection mode {mode!r}")
    if override is not None:
        return WorkflowDecision(override, b, basis, threshold)
    chosen = Workflow.RLE_VLE if b <= threshold else Workflow.HUFFMAN
    return WorkflowDecision(chosen, b, basis, threshold)
