"""a1 — the partition plan (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Paper anchors:
  P:279 (§4.2.1)  "split the entire checkpoint into multiple parts, transferring
                  a portion at each step"; parts A, B, C ride steps N+1..N+3 and
                  "the gradients corresponding to the existing checkpoints"
                  (G_A^1, G_AB^2) ride along.
  SPEC S:131-139  make_parts: K balanced contiguous parts, remainder to the
                  earliest parts; (P=10, K=3) -> [0,4), [4,7), [7,10).

Reading R11: balance over U = ceil(n/A) units of A elements,
remainder units to the earliest parts, the last part absorbs the partial tail
unit. A=1 is SPEC's rule.
"""

from __future__ import annotations


def make_parts(n: int, K: int, A: int = 1):
    """Return K half-open ranges [(lo_1, hi_1), ..., (lo_K, hi_K)] tiling [0, n)."""
    if n < 1 or K < 1 or A < 1:
        raise ValueError("n, K, A must be >= 1")
    U = -(-n // A)  # ceil
    if K > U:
        raise ValueError("K must not exceed the number of A-element units")
    base, rem = divmod(U, K)
    parts = []
    lo_unit = 0
    for i in range(1, K + 1):
        units = base + (1 if i <= rem else 0)
        hi_unit = lo_unit + units
        parts.append((min(lo_unit * A, n), min(hi_unit * A, n)))
        lo_unit = hi_unit
    return parts


def grad_prefix(parts, i: int) -> int:
    """Session step i (1-based) records G(t0+i)[0:hi_i] for i < K; step K records nothing."""
    K = len(parts)
    return parts[i - 1][1] if i < K else 0


def slot_bytes(parts, i: int) -> int:
    """V_i: bytes session step i moves device->host: 12*|P_i| + 2*prefix_i."""
    lo, hi = parts[i - 1]
    return 12 * (hi - lo) + 2 * grad_prefix(parts, i)


def session_bytes(parts) -> int:
    """Total D2H bytes of one session: sum_i V_i."""
    return sum(slot_bytes(parts, i) for i in range(1, len(parts) + 1))


# ---- the transfer-balanced plan (reading R17) -----------------------------------
# P:279 splits the checkpoint into parts that ride consecutive steps with "the gradients
# corresponding to the existing checkpoints"; the paper does not fix the part sizes (S:131 makes
# them equal). Step i moves V_i = 12 |P_i| + 2 hi_i bytes (i < K) and V_K = 12 |P_K|, so with equal
# parts the last gradient-carrying step is the largest, V_max ~ (10 + 2K) n / K. The balanced plan
# instead picks the contiguous parts (boundaries on A-element units) that make the largest V_i as
# small as the rule below finds: for a byte budget V, fill parts 1..K-1 greedily, each taking the
# most whole units u with 12 A u + 2 A (H + u) <= V (at least one unit, and one unit left for every
# later part), the last part taking the rest; the plan is the greedy fill at the smallest V (binary
# search over integers, [0, 14 n]) whose fill keeps every V_i <= V. If that is not strictly better
# than the equal plan, the equal plan is kept.


def max_slot_bytes(parts) -> int:
    """V_max = max_i V_i of a plan."""
    return max(slot_bytes(parts, i) for i in range(1, len(parts) + 1))


def _greedy_fill(n: int, K: int, A: int, V: int):
    U = -(-n // A)
    H = 0  # units covered by parts 1..i
    bounds = []
    for i in range(1, K):
        cap = (V - 2 * A * H) // (14 * A) if V >= 2 * A * H else 0
        u = min(max(cap, 1), U - H - (K - i))
        H += u
        bounds.append(H)
    parts = []
    lo = 0
    for h in bounds:
        parts.append((lo, h * A))
        lo = h * A
    parts.append((lo, n))
    return parts


def make_parts_balanced(n: int, K: int, A: int = 1):
    """The transfer-balanced plan: K contiguous parts tiling [0, n) (see the comment above)."""
    if n < 1 or K < 1 or A < 1:
        raise ValueError("n, K, A must be >= 1")
    U = -(-n // A)
    if K > U:
        raise ValueError("K must not exceed the number of A-element units")
    equal = make_parts(n, K, A)
    if K == 1:
        return equal
    lo, hi = 0, 14 * n  # any plan has V_i <= 12 n + 2 n, so the fill at 14 n qualifies
    while lo < hi:
        mid = (lo + hi) // 2
        if max_slot_bytes(_greedy_fill(n, K, A, mid)) <= mid:
            hi = mid
        else:
            lo = mid + 1
    parts = _greedy_fill(n, K, A, lo)
    return parts if max_slot_bytes(parts) < max_slot_bytes(equal) else equal
