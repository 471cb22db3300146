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
