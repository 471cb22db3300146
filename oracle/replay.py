"""O2 — plain K-step partitioned capture + gradient-assisted replay
(TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Paper anchors, in the order the algorithm follows them:
  P:279 (§4.2.1)  "we begin the checkpoint operation after Step N ... divided
                  into three parts: A, B, and C ... overlap with training in
                  Step N+1, N+2, and N+3 ... we also need to transfer the
                  gradients corresponding to the existing checkpoints to the
                  CPU at each step (G_A^1 and G_AB^2)".
  P:345 (§4.3.1)  "For checkpoint version 1 of part A transferred at Step N+1,
                  gradients of part A computed in Steps N+1 and N+2 are used to
                  update checkpoint version 3 ... part B transferred at Step
                  N+2 is updated with part B's gradients computed at Step N+2
                  ... equivalent to directly transferring the checkpoint from
                  Step N+3 to CPU memory."

Generalised to K parts (readings R1-R3): session step i = training
step t0+i (i = 1..K) captures part i at S(t0+i-1) (before update t0+i) and, for
i < K, records G(t0+i) restricted to parts 1..i = the prefix [0, hi_i). The
replay brings each part j < K from S(t0+j-1) to S(T), T = t0+K-1, by applying
updates t0+j .. t0+K-1 in ascending order.
"""

from __future__ import annotations

import numpy as np

from .adamw import adamw_update
from .partition import make_parts


def capture_session(p0, m0, v0, grads, recs, parts):
    """Run session steps i = 1..K of live training from S(t0) and capture.

    grads[i-1] / recs[i-1] drive update t0+i. Returns (cap, glog, live) where
    cap[i-1] = (p, m, v) of part i at S(t0+i-1), glog[i-1] = G(t0+i)[0:hi_i]
    (i < K), and live = the live state after update t0+K.
    """
    K = len(parts)
    p, m, v = (np.array(x, dtype=np.float32) for x in (p0, m0, v0))
    cap, glog = [], []
    for i in range(1, K + 1):
        lo, hi = parts[i - 1]
        cap.append((p[lo:hi].copy(), m[lo:hi].copy(), v[lo:hi].copy()))   # version S(t0+i-1)
        if i < K:
            glog.append(np.array(grads[i - 1][0:hi], dtype=np.uint16))     # G(t0+i) on parts 1..i
        p, m, v, _ = adamw_update(p, m, v, grads[i - 1], recs[i - 1])     # update t0+i
    return cap, glog, (p, m, v)


def assemble(cap):
    """Concatenate the K captured parts into the (stale) host checkpoint."""
    p = np.concatenate([c[0] for c in cap])
    m = np.concatenate([c[1] for c in cap])
    v = np.concatenate([c[2] for c in cap])
    return p, m, v


def replay(cap, glog, recs, parts):
    """Gradient-assisted replay: every part j < K is brought to S(t0+K-1).

    for j in 1..K-1:  for e in P_j:  for i in j..K-1:
        ckpt[e] = adamw(ckpt[e], glog[i][e], StepRecord(t0+i))
    (vectorised over e within P_j; the per-element op sequence is exactly that.)
    """
    K = len(parts)
    p, m, v = assemble(cap)
    for j in range(1, K):
        lo, hi = parts[j - 1]
        pj, mj, vj = p[lo:hi], m[lo:hi], v[lo:hi]
        for i in range(j, K):
            pj, mj, vj, _ = adamw_update(pj, mj, vj, glog[i - 1][lo:hi], recs[i - 1])
        p[lo:hi], m[lo:hi], v[lo:hi] = pj, mj, vj
    return p, m, v


def replay_streaming(cap, glog, recs, parts):
    """Streaming form of the same replay (SURVEY §8(a) a5 "Streaming"; P:345's updates applied as
    the slices arrive): the parts land in order; once part i and G(t0+i)[0:hi_i] are on the host
    (i < K), update t0+i is applied to the whole prefix [0, hi_i) = parts 1..i, which are then all
    at S(t0+i). Element e of part j receives updates t0+j .. t0+K-1 in ascending order, the batch
    order, so the result must equal replay() bit for bit.
    """
    K = len(parts)
    p, m, v = assemble(cap)                     # part i's bytes are only read after it "lands"
    for i in range(1, K):
        hi = parts[i - 1][1]
        p[:hi], m[:hi], v[:hi], _ = adamw_update(p[:hi], m[:hi], v[:hi], glog[i - 1][:hi], recs[i - 1])
    return p, m, v


def oracle_session(p0, m0, v0, grads, recs, K: int, A: int = 1):
    """Full O2 on [0, n): plan, capture over K steps, replay. Returns (ckpt, cap, glog, parts, live)."""
    n = len(p0)
    parts = make_parts(n, K, A)
    cap, glog, live = capture_session(p0, m0, v0, grads, recs, parts)
    return replay(cap, glog, recs, parts), cap, glog, parts, live
