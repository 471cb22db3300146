"""Pins of the oracle's partition plan and partitioned replay (-m "not gpu").

The paper's invariant ("equivalent to directly transferring the
checkpoint from Step N+3"): the replayed checkpoint equals the synchronous
snapshot S(T), T = t0+K-1. Checked by brute force over EVERY contiguous
partition of tiny vectors, over SPEC's sweep sizes, and on the paper's
K=3 trace (P:279 G_A^1 / G_AB^2).
"""

import itertools

import numpy as np
import pytest

from oracle import (adamw_update, make_step_record, trajectory, make_parts, grad_prefix,
                    session_bytes, slot_bytes, capture_session, replay, replay_streaming, oracle_session)
import gockpt_inputs as gi

HP = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


def recs_for(t0, K, skips=()):
    out, t = [], 0
    # bias-correction count: non-skipped updates up to and including step s (reading R8)
    for s in range(1, t0 + K + 1):
        sk = s in skips
        if not sk:
            t += 1
        if s > t0:
            out.append(make_step_record(t=t, lr=1e-3 * (1 + 0.01 * s), grad_scale=1.0 if s % 3 else 0.5,
                                        skip=sk, **HP))
    return out


def grads_for(seed, t0, K, n, mode):
    return [gi.grad_bits(seed, t0 + i, n, mode=mode) for i in range(1, K + 1)]


def states_equal(a, b):
    return all(np.array_equal(x.view(np.uint32), y.view(np.uint32)) for x, y in zip(a, b))


# ---------------------------------------------------------------- make_parts
def test_make_parts_spec_examples():
    assert make_parts(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert make_parts(10, 1) == [(0, 10)]
    assert make_parts(7, 7) == [(i, i + 1) for i in range(7)]
    with pytest.raises(ValueError):
        make_parts(5, 6)


@pytest.mark.parametrize("n,K,A", [(2 ** 20, 4, 1024), (1_000_003, 4, 1024), (124_439_808, 8, 1024),
                                   (5000, 5, 1024), (3 * 1024 + 1, 4, 1024), (1, 1, 1024)])
def test_make_parts_aligned_properties(n, K, A):
    parts = make_parts(n, K, A)
    assert parts[0][0] == 0 and parts[-1][1] == n
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c and a < b
        assert b % A == 0                      # interior boundaries are A-aligned
    units = [-(-(hi - lo) // A) for lo, hi in parts]
    assert max(units) - min(units) <= 1        # balanced over A-element units
    assert units == sorted(units, reverse=True)  # remainder to the earliest parts


def test_byte_counts_closed_form():
    # SURVEY §8 sizes: with equal parts, session D2H = 12n + sum_{i<K} 2 hi_i = n(11+K)
    for n, K in [(2 ** 20, 4), (8 * 1024 * 10, 8), (16 * 64, 16)]:
        parts = make_parts(n, K, 64)
        assert session_bytes(parts) == n * (11 + K)
        assert slot_bytes(parts, K) == 12 * n // K
        assert max(slot_bytes(parts, i) for i in range(1, K + 1)) == slot_bytes(parts, K - 1) if K > 1 else True
        assert slot_bytes(parts, K - 1) == (10 + 2 * K) * n // K if K > 1 else True
    parts = make_parts(10, 3)
    assert [grad_prefix(parts, i) for i in (1, 2, 3)] == [4, 7, 0]


# ---------------------------------------------------------------- the paper's K=3 trace
def test_k3_trace_versions_and_slices():
    n, t0, K, seed = 10, 5, 3, 42
    p0, m0, v0 = gi.warm_state(seed, n)
    recs = recs_for(t0, K)
    grads = grads_for(seed, t0, K, n, gi.GRAD_LLM)
    S = trajectory(p0, m0, v0, grads, recs)          # S[k] = S(t0+k)
    parts = make_parts(n, K)
    cap, glog, live = capture_session(p0, m0, v0, grads, recs, parts)
    # ledger {A: S(N), B: S(N+1), C: S(N+2)}  (SPEC S:175 with N = t0)
    for i, (lo, hi) in enumerate(parts):
        assert states_equal(cap[i], tuple(x[lo:hi] for x in S[i]))
    # slices {G(N+1) on A, G(N+2) on A u B}; no G(N+3)  ("G_A^1 and G_AB^2")
    assert len(glog) == 2
    assert np.array_equal(glog[0], grads[0][: parts[0][1]])
    assert np.array_equal(glog[1], grads[1][: parts[1][1]])
    assert states_equal(live, S[3])
    # target version S(N+2) (K=3 -> S(N+2), "checkpoint version 3")
    assert states_equal(replay(cap, glog, recs, parts), S[K - 1])


def test_k1_is_identity():
    n, t0, seed = 17, 3, 7
    p0, m0, v0 = gi.warm_state(seed, n)
    ck, cap, glog, parts, _ = oracle_session(p0, m0, v0, grads_for(seed, t0, 1, n, gi.GRAD_LLM),
                                             recs_for(t0, 1), K=1)
    assert glog == [] and parts == [(0, n)]
    assert states_equal(ck, (p0, m0, v0))


# ---------------------------------------------------------------- brute force, every composition
def compositions(n, K):
    for cuts in itertools.combinations(range(1, n), K - 1):
        b = (0,) + cuts + (n,)
        yield [(b[i], b[i + 1]) for i in range(K)]


@pytest.mark.parametrize("mode", [gi.GRAD_UNIFORM, gi.GRAD_LLM])
@pytest.mark.parametrize("t0", [0, 1, 5])
def test_brute_force_every_partition(mode, t0):
    count = 0
    for seed in (42, 7, 1, 2, 3):
        for n in range(1, 10):
            p0, m0, v0 = gi.warm_state(seed, n) if t0 else gi.cold_state(seed, n)
            for K in range(1, n + 1):
                recs = recs_for(t0, K)
                grads = grads_for(seed, t0, K, n, mode)
                target = trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]   # O1: S(t0+K-1)
                for parts in compositions(n, K):
                    cap, glog, _ = capture_session(p0, m0, v0, grads, recs, parts)
                    assert states_equal(replay(cap, glog, recs, parts), target), (seed, n, K, parts)
                    # the streaming order (slices applied as they land) reaches the same bytes
                    assert states_equal(replay_streaming(cap, glog, recs, parts), target), (seed, n, K, parts)
                    count += 1
    assert count == 5 * (2 ** 9 - 1)


def test_skipped_steps_inside_session():
    n, t0, K, seed = 9, 4, 4, 3
    p0, m0, v0 = gi.warm_state(seed, n)
    recs = recs_for(t0, K, skips={t0 + 2})
    assert recs[1].skip and recs[2].t == recs[0].t + 1     # a skip does not advance t
    grads = grads_for(seed, t0, K, n, gi.GRAD_LLM)
    target = trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]
    for parts in compositions(n, K):
        cap, glog, _ = capture_session(p0, m0, v0, grads, recs, parts)
        assert states_equal(replay(cap, glog, recs, parts), target)


# ---------------------------------------------------------------- SPEC-sized sweep
@pytest.mark.parametrize("n", [64, 1000, 100000])
@pytest.mark.parametrize("mode", [gi.GRAD_UNIFORM, gi.GRAD_LLM])
def test_spec_sweep(n, mode):
    for K in range(1, 9):
        for seed in (42, 7):
            t0 = 10
            p0, m0, v0 = gi.warm_state(seed, n)
            recs = recs_for(t0, K)
            grads = grads_for(seed, t0, K, n, mode)
            target = trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]
            ck, *_ = oracle_session(p0, m0, v0, grads, recs, K=K, A=1 if n < 1000 else 16)
            assert states_equal(ck, target), (n, K, seed)


def test_k_independence_at_fixed_target():
    # Reading R11: S(T) is independent of K and of the partition for fixed T (elementwise update)
    n, T, seed = 1000, 12, 1
    results = []
    for K in (1, 2, 3, 5, 8):
        t0 = T - K + 1
        recs = recs_for(t0, K)
        # the same absolute gradients G(t) for every K: regenerate the trajectory from S(0)
        p, m, v = gi.cold_state(seed, n)
        pre = recs_for(0, t0)
        for s in range(1, t0 + 1):
            p, m, v, _ = adamw_update(p, m, v, gi.grad_bits(seed, s, n), pre[s - 1])
        ck, *_ = oracle_session(p, m, v, grads_for(seed, t0, K, n, gi.GRAD_LLM), recs, K=K, A=8)
        results.append(ck)
    for r in results[1:]:
        assert states_equal(r, results[0])


# ---------------------------------------------------------------- negative controls
def test_negative_controls_detected():
    n, t0, K, seed = 4096, 10, 4, 42
    p0, m0, v0 = gi.warm_state(seed, n)
    recs = recs_for(t0, K)
    grads = grads_for(seed, t0, K, n, gi.GRAD_LLM)
    target = trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]
    parts = make_parts(n, K, 64)
    cap, glog, _ = capture_session(p0, m0, v0, grads, recs, parts)
    assert states_equal(replay(cap, glog, recs, parts), target)
    # (1) no replay
    from oracle import assemble
    assert not states_equal(assemble(cap), target)
    # (2) a dropped gradient slice (zeros instead of G)
    bad = [g.copy() for g in glog]
    bad[1][:] = 0
    assert not states_equal(replay(cap, bad, recs, parts), target)
    # (3) post-update capture misreading: capture part i at S(t0+i)
    S = trajectory(p0, m0, v0, grads, recs)
    cap_post = [tuple(x[lo:hi] for x in S[i + 1]) for i, (lo, hi) in enumerate(parts)]
    assert not states_equal(replay(cap_post, glog, recs, parts), target)
    # (4) a flipped byte in a captured part
    flip = [tuple(x.copy() for x in c) for c in cap]
    flip[0][1].view(np.uint8)[5] ^= 0x10
    assert not states_equal(replay(flip, glog, recs, parts), target)
    # (5) steps replayed in the wrong order
    rev = list(reversed(glog))
    rev = [np.concatenate([r, np.zeros(len(glog[-1]) - len(r), np.uint16)])[: len(g)] for r, g in zip(rev, glog)]
    assert not states_equal(replay(cap, rev, recs, parts), target)
