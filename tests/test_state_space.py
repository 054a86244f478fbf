"""NEXT-2: drift PMF and state-space sizing exported by the C ABI
(bsidmap_drift_pmf / bsidmap_drift_limits / bsidmap_state_space; host code, no GPU).
Pinned by brute-force enumeration of per-bit channel events, SPEC's worked values
(tests/golden/spec_examples.txt) and the closed-form mean of the drift."""
import os

import numpy as np
import pytest

from paper_1802_08483_b200 import drift_limits, drift_pmf, state_space
from tests import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


@pytest.mark.parametrize("T,Pi,Pd", [(1, 0.1, 0.1), (2, 0.2, 0.05), (3, 0.05, 0.3), (4, 0.1, 0.1), (5, 0.0, 0.2)])
def test_drift_pmf_equals_enumeration(T, Pi, Pd):
    kmax = 10 if T <= 3 else 8 if T == 4 else 5
    ref = brute.drift_enum(T, Pi, Pd, kmax=kmax)
    # the enumeration truncates a bit's insertions at kmax: drifts m <= kmax - T are exact
    lo, hi = -T, kmax - T if Pi > 0 else T
    got = drift_pmf(T, Pi, Pd, lo, hi)
    for m in range(lo, hi + 1):
        assert got[m - lo] == pytest.approx(ref.get(m, 0.0), rel=1e-9, abs=1e-15)


def test_drift_pmf_spec_values():
    for line in open(GOLDEN):
        line = line.split("#")[0].split()
        if not line or line[0] != "drift_pmf":
            continue
        T, Pi, Pd = int(line[1]), float(line[2]), float(line[3])
        got = drift_pmf(T, Pi, Pd, -T, T + 3)
        for item in line[4].split(","):
            m, v = item.split(":")
            assert got[int(m) + T] == pytest.approx(float(v), rel=1e-12)


def test_drift_mean_and_mass():
    T, Pi, Pd = 200, 0.05, 0.03
    lo, hi = -T, 200
    p = drift_pmf(T, Pi, Pd, lo, hi)
    m = np.arange(lo, hi + 1)
    assert p.sum() == pytest.approx(1.0, abs=1e-12)
    assert (p * m).sum() == pytest.approx(T * (Pi - Pd) / (1 - Pi), rel=1e-10)


CASES = [(10, 0.01, 0.01, 1e-10), (1000, 0.1, 0.1, 1e-10), (120000, 0.02, 0.02, 1e-10), (50, 0.2, 0.05, 1e-6),
         (2100, 1e-3, 1e-3, 1e-10), (12, 0.02, 0.02, 1e-10), (7, 0.01, 0.01, 1e-10)]


def _pmf(T, Pi, Pd):
    W = 4000
    lo = -min(T, W)
    return np.arange(lo, W + 1), drift_pmf(T, Pi, Pd, lo, W)


@pytest.mark.parametrize("T,Pi,Pd,Pr", CASES)
def test_limits_cover_and_are_minimal(T, Pi, Pd, Pr):
    """the interval contains 0, its excluded mass is < Pr, and it is minimal --
    shrinking either end (where it is not already 0) breaks the coverage."""
    lo, hi = drift_limits(T, Pi, Pd, Pr)
    assert -T <= lo <= 0 <= hi
    m, p = _pmf(T, Pi, Pd)
    excl = lambda a, b: p[m < a].sum() + p[m > b].sum()
    assert excl(lo, hi) < Pr
    if lo < 0:
        assert excl(lo + 1, hi) >= Pr
    if hi > 0:
        assert excl(lo, hi - 1) >= Pr


@pytest.mark.parametrize("T,Pi,Pd,Pr", CASES)
def test_limits_equal_greedy_growth_by_hand(T, Pi, Pd, Pr):
    """The growth order of SPEC S:62 replayed on the exported PMF with plain sums (no tail
    bookkeeping): extend the side with more excluded mass, ties to the positive side."""
    m, p = _pmf(T, Pi, Pd)
    lo = hi = 0
    while p[m < lo].sum() + p[m > hi].sum() >= Pr:
        if p[m > hi].sum() >= p[m < lo].sum():
            hi += 1
        else:
            lo -= 1
    assert drift_limits(T, Pi, Pd, Pr) == (lo, hi)
    import bsidgen
    assert bsidgen.drift_limits(T, Pi, Pd, Pr) == (lo, hi)


def test_limits_noiseless_and_zero_length():
    assert drift_limits(0, 0.1, 0.1) == (0, 0)       # S_0 = 0
    assert drift_limits(500, 0.0, 0.0) == (0, 0)     # SPEC: pi = pd = 0 -> (0, 0)
    lo, hi = drift_limits(40, 0.0, 0.05)             # deletions only: the drift is never positive
    assert hi == 0 and lo < 0


@pytest.mark.parametrize("T,Pi,Pd,Pr", CASES)
def test_tail_rule_covers_and_is_minimal_per_tail(T, Pi, Pd, Pr):
    """The per-tail rule (bsidmap_drift_limits_tails): each tail <= Pr/2, one state tighter on
    either side exceeds Pr/2 (unless clamped at 0 / -T); never tighter than the greedy rule's sum."""
    lo, hi = drift_limits(T, Pi, Pd, Pr, rule="tails")
    assert -T <= lo <= 0 <= hi
    m, p = _pmf(T, Pi, Pd)
    assert p[m < lo].sum() <= Pr / 2 and p[m > hi].sum() <= Pr / 2
    if lo < 0 and lo > -T:
        assert p[m < lo + 1].sum() > Pr / 2
    if hi > 0:
        assert p[m > hi - 1].sum() > Pr / 2
    glo, ghi = drift_limits(T, Pi, Pd, Pr)
    assert ghi - glo <= hi - lo


def test_state_space_of_the_baseline_configs():
    # m_n from T = n, m_tau from T = n N widened to contain m_n (DESIGN.md section 4 table)
    table = {(7, 10, 0.01): ((-5, 6), (-10, 11)), (10, 100, 0.01): ((-6, 6), (-30, 31)),
             (8, 500, 0.05): ((-7, 11), (-132, 134)), (10, 1000, 0.1): ((-10, 15), (-303, 307)),
             (12, 10000, 0.02): ((-7, 8), (-452, 453))}
    for (n, N, p), want in table.items():
        assert state_space(n, N, p, p) == want
