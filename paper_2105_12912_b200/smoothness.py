"""Workflow selection (mirrors P/smoothness.py:26-37, 111-136).

The 1.09-bit rule: a stream expected to Huffman-code at or below
RLE_THRESHOLD_BITS bits/symbol goes to RLE + VLE.  Exact mode uses the true
average code length of the device-built code book (K2 returns sum(c*len) and
the total; the division is done here exactly as numpy does it).  Estimate
mode evaluates the entropy + redundancy bracket on the cap-bin histogram --
host arithmetic on a few KB, kept on the host so the floats are bit-identical
with numpy (the entropy bounds are host-side by design).

``analyze`` / ``sample_madogram`` (P/smoothness.py:40-108, 139-188) are
profiling tools outside the compress path.  The element
work (prequantization, K1 codes, the histogram) runs on the GPU; the pairs
are drawn on the host with numpy's PCG64 exactly as the reference draws them
(same seed -> same pairs), only the sampled elements are gathered from the
device, and the per-distance means are the reference's numpy arithmetic.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .errors import DataError

RLE_THRESHOLD_BITS = 1.09

#: Largest pair separation sampled by default (P/smoothness.py:29).
DEFAULT_DMAX = 200


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


@dataclass(frozen=True)
class MadogramReport:
    """Per-distance mean variance of sampled pairs (P/smoothness.py:40-50)."""

    kind: str  # "binary" | "absolute"
    distances: np.ndarray  # int64, measured separations, ascending
    variance: np.ndarray  # float64, mean v(d) per measured distance
    sample_count: int
    seed: int
    roughness: float  # unweighted mean of v(d)
    smoothness: float | None  # 1 - roughness, binary kind only


def default_sample_count(count: int, dmax: int = DEFAULT_DMAX) -> int:
    """At least 10 samples per distance, capped by the data size (P/smoothness.py:63-65)."""
    return max(10 * dmax, min(count // 10, 100 * dmax))


def _gather_f64(values, idx: np.ndarray) -> np.ndarray:
    """values[idx] as float64 -- a device gather when values is a CUDA tensor."""
    try:
        import torch

        if isinstance(values, torch.Tensor):
            t = torch.from_numpy(idx.astype(np.int64)).to(values.device)
            return values.reshape(-1)[t].to(torch.float64).cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(values).reshape(-1)[idx].astype(np.float64)


def sample_madogram(values, kind: str = "binary", n: int | None = None, dmax: int = DEFAULT_DMAX,
                    seed: int = 0) -> MadogramReport:
    """v(d) for d in [1, dmax] from n random pairs (a, a+d), P/smoothness.py:68-108.

    The draws (and the redraw of pairs that fall off the end) are the
    reference's, so a given seed samples the same pairs; `values` may be a
    numpy array or a CUDA tensor (only the sampled elements leave the device)."""
    if kind not in ("binary", "absolute"):
        raise DataError(f"unknown madogram kind {kind!r}")
    count = int(values.numel()) if hasattr(values, "numel") else int(np.asarray(values).size)
    if count < 2:
        raise DataError("madogram needs at least 2 elements")
    if n is None:
        n = default_sample_count(count, dmax)
    if n < 1:
        raise DataError("sample count must be >= 1")
    rng = np.random.default_rng(seed)
    sums = np.zeros(dmax + 1)
    hits = np.zeros(dmax + 1, np.int64)
    remaining = n
    while remaining:
        a = rng.integers(0, count, size=remaining)
        d = rng.integers(1, dmax + 1, size=remaining)
        ok = a + d < count
        a, d = a[ok], d[ok]
        za = _gather_f64(values, a)
        zb = _gather_f64(values, a + d)
        diff = zb != za if kind == "binary" else np.abs(zb - za)
        np.add.at(sums, d, diff)
        np.add.at(hits, d, 1)
        remaining -= int(ok.sum())
    measured = np.flatnonzero(hits)
    v = sums[measured] / hits[measured]
    roughness = float(v.mean())
    smooth = 1.0 - roughness if kind == "binary" else None
    return MadogramReport(kind, measured.astype(np.int64), v, n, seed, roughness, smooth)


@dataclass(frozen=True)
class AnalysisRecord:
    """Madogram profiles of both stages + histogram stats + decision (P/smoothness.py:139-163)."""

    reports: tuple  # ((stage, MadogramReport), ...)
    entropy: object  # EntropyReport
    decision: WorkflowDecision
    smoothness: float  # binary smoothness of the prequantized data

    def to_csv(self) -> str:
        lines = ["stage,kind,distance,variance"]
        for stage, rep in self.reports:
            lines += [f"{stage},{rep.kind},{d},{v:.9g}" for d, v in zip(rep.distances, rep.variance)]
        e, dec = self.entropy, self.decision
        b_exact = float("nan") if e.b_exact is None else e.b_exact
        lines += [f"# H={e.entropy:.9g}", f"# p1={e.p1:.9g}", f"# b_lo={e.b_lo:.9g}",
                  f"# b_hi={e.b_hi:.9g}", f"# b_exact={b_exact:.9g}",
                  f"# smoothness={self.smoothness:.9g}", f"# decision={dec.chosen.name}"]
        return "\n".join(lines) + "\n"


def analyze(field, cfg, chunk=None, dmax: int = DEFAULT_DMAX, seed: int = 0,
            mode: str = "exact") -> AnalysisRecord:
    """Compressibility profile before and after quantization (P/smoothness.py:166-188):
    prequant (GPU) -> K1 codes in grid order (GPU) -> madograms of both stages
    (pairs gathered from the device) -> histogram stats and the workflow decision."""
    from .codebook import Codebook, entropy_report
    from .grid import ChunkSpec
    from .quantize import prequantize_device, quant_grid_device

    chunk = chunk or ChunkSpec.default_for(field.dims.ndim)
    pre = prequantize_device(field, cfg)
    codes, counts = quant_grid_device(pre, field.dims, cfg, chunk)
    reports = []
    for stage, data in (("prequant", pre), ("quant-code", codes)):
        for kind in ("binary", "absolute"):
            reports.append((stage, sample_madogram(data, kind, dmax=dmax, seed=seed)))
    book = Codebook.from_counts(counts)
    rep = entropy_report(counts, book)
    decision = select_workflow(counts, mode=mode)
    return AnalysisRecord(tuple(reports), rep, decision, float(reports[0][1].smoothness or 0.0))
