"""Pins of the oracle's transfer-balanced plan (oracle.partition.make_parts_balanced, R17).

The plan is defined by a rule (greedy fill at the smallest byte budget, integer binary search);
these tests pin it to what that rule is meant to achieve, computed independently of it:
  - it tiles [0, n) with K non-empty contiguous parts on A-element boundaries;
  - its largest per-step transfer V_max equals the brute-force minimum over EVERY contiguous
    unit-aligned K-part partition (all compositions of the U units) for small U, K;
  - it is never worse than the equal plan and matches the continuous optimum of the
    balance equations for large n;
  - a hand-worked example (n = 10, K = 3, A = 1).
"""
import itertools
import math

import pytest

from oracle.partition import make_parts, make_parts_balanced, max_slot_bytes, slot_bytes


def _tiles(parts, n, K, A):
    assert len(parts) == K
    assert parts[0][0] == 0 and parts[-1][1] == n
    for (a, b), (c, _) in zip(parts, parts[1:]):
        assert b == c
    for lo, hi in parts:
        assert hi > lo
        assert lo % A == 0
    for lo, hi in parts[:-1]:
        assert hi % A == 0


def _brute_min_vmax(n, K, A):
    U = -(-n // A)
    best = None
    for cuts in itertools.combinations(range(1, U), K - 1):
        b = (0,) + cuts + (U,)
        parts = [(min(b[i] * A, n), min(b[i + 1] * A, n)) for i in range(K)]
        # V_i written out from its definition (part i + the gradient prefix of parts 1..i)
        v = max(12 * (hi - lo) + (2 * hi if i < K - 1 else 0) for i, (lo, hi) in enumerate(parts))
        best = v if best is None else min(best, v)
    return best


def test_hand_worked_n10_k3():
    # V_1 = 14 p1, V_2 = 14 p2 + 2 p1, V_3 = 12 p3 with p1 + p2 + p3 = 10. V <= 47 forces p1 <= 3,
    # p2 <= 2 (p1 + p2 <= 5) and p3 <= 3: infeasible; V = 48 is met by (3, 3, 4): 42, 48, 48.
    parts = make_parts_balanced(10, 3, 1)
    assert parts == [(0, 3), (3, 6), (6, 10)]
    assert [slot_bytes(parts, i) for i in (1, 2, 3)] == [42, 48, 48]
    assert max_slot_bytes(make_parts(10, 3, 1)) == 56  # equal plan (S:137 example): 48+8, 36+14, 36


@pytest.mark.parametrize("A", [1, 3])
def test_brute_force_optimal_small(A):
    cases = 0
    for U in range(1, 14):
        for tail in ([0] if A == 1 else [0, 2]):
            n = U * A - tail
            if n < 1:
                continue
            for K in range(1, min(U, 7) + 1):
                parts = make_parts_balanced(n, K, A)
                _tiles(parts, n, K, A)
                assert max_slot_bytes(parts) == _brute_min_vmax(n, K, A), (n, K, A)
                cases += 1
    assert cases > 60


@pytest.mark.parametrize("n,K,A", [(124_439_808, 8, 1024), (842_301_952, 8, 1024), (3_253_966_336, 16, 1024),
                                   (6_507_932_160, 16, 1024), (1 << 20, 4, 1024), (1_000_003, 64, 8),
                                   (5000, 2, 1), (4096, 4096, 1)])
def test_never_worse_than_equal_and_tiles(n, K, A):
    b, e = make_parts_balanced(n, K, A), make_parts(n, K, A)
    _tiles(b, n, K, A)
    assert max_slot_bytes(b) <= max_slot_bytes(e)


@pytest.mark.parametrize("K", [2, 4, 8, 16, 32])
def test_continuous_optimum_large_n(K):
    # Real-valued balance: V = 14 p_1 = 14 p_i + 2 H_{i-1} (i < K) = 12 p_K gives
    # H_i = (V/2)(1 - (6/7)^i) and n = H_{K-1} + V/12, so V*/n = 1 / ((1 - (6/7)^(K-1))/2 + 1/12).
    n, A = 3_253_966_336, 1024
    vstar = n / ((1 - (6 / 7) ** (K - 1)) / 2 + 1 / 12)
    v = max_slot_bytes(make_parts_balanced(n, K, A))
    assert v >= vstar * (1 - 1e-9)  # integer parts cannot beat the relaxation
    assert v <= vstar + 14 * A * 2  # within two units of rounding
    # and the equal plan's V_max is (10 + 2K) n / K up to rounding: the balanced one is smaller
    assert v < (10 + 2 * K) * n / K
