"""The paper's operator performance model (the formulas of ``lqcdlab.perf``,
perf.py:47-99), kept so code that reports against the reference's model runs
unchanged.  The B200 path itself is measured against the HBM roofline with the
compulsory-byte count of ``dirac.compulsory_bytes_per_site``; these
are the CPU paper's counts (2574 b flop and (168 b + 114) complex values moved
per site, dirac.py:43-48)."""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .dirac import BYTES_PER_VALUE, FLOPS_PER_SITE_RHS, VALUES_PER_SITE_FIXED, VALUES_PER_SITE_RHS


def arithmetic_intensity(b: int) -> Fraction:
    """Flop per byte of one b-rhs apply: 2574 b / ((168 b + 114) * 16) (perf.py:64-71)."""
    if b < 1:
        raise ValueError("b must be >= 1")
    return Fraction(FLOPS_PER_SITE_RHS * b, (VALUES_PER_SITE_RHS * b + VALUES_PER_SITE_FIXED) * BYTES_PER_VALUE)


def theoretical_perf(bw: float, b: int) -> float:
    """Bandwidth-bound flop/s ceiling at bw bytes/s (perf.py:74-78)."""
    if bw <= 0:
        raise ValueError("bandwidth must be positive")
    return bw * float(arithmetic_intensity(b))


def arch_efficiency(measured: float, theoretical: float) -> float:
    """measured / theoretical (perf.py:81-86)."""
    if theoretical <= 0:
        raise ValueError("theoretical performance must be positive")
    if measured < 0:
        raise ValueError("measured performance must be nonnegative")
    return measured / theoretical


def read_write_ratio(b: int) -> Fraction:
    """(204 b + 330) : 204 b read-to-write traffic of the operator (perf.py:95-99)."""
    if b < 1:
        raise ValueError("b must be >= 1")
    return Fraction(204 * b + 330, 204 * b)


@dataclass
class CounterSample:
    """Cache refill / writeback counters of one measurement (perf.py:47-61)."""

    l2_refill: int
    l2_writeback: int
    cycles: int
    frequency: float
    cache_line: int = 256
    ranks: int = 1

    def __post_init__(self) -> None:
        if min(self.l2_refill, self.l2_writeback) < 0:
            raise ValueError("counters must be nonnegative")
        if self.cycles <= 0:
            raise ValueError("cycles must be positive")


def effective_bandwidth(sample: CounterSample) -> float:
    """Bytes/s implied by refill + writeback lines over the sampled cycles (perf.py:89-92)."""
    lines = sample.l2_refill + sample.l2_writeback
    return lines * sample.cache_line * sample.frequency / sample.cycles * sample.ranks
