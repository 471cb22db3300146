"""Property-based checks (hypothesis, -m "not gpu"): for random shard sizes, K, alignments,
skipped steps, grad scales and learning-rate schedules, the library's host replay equals the
oracle's O2 and O1 bit for bit, and its plan equals the oracle's."""

import numpy as np
from hypothesis import given, settings, strategies as st, HealthCheck

import gockpt_inputs as gi
import oracle

HP = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


def _G():
    from paper_2511_07035_b200 import build as gbuild
    gbuild.build()
    import paper_2511_07035_b200 as G
    return G


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(n=st.integers(1, 5000), K=st.integers(1, 12), A=st.sampled_from([1, 8, 64, 1024]))
def test_plan_matches_oracle(n, K, A):
    G = _G()
    U = -(-n // A)
    if K > U:
        return
    assert G.plan_parts(n, K, A) == oracle.make_parts(n, K, A)


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(n=st.integers(1, 3000), K=st.integers(1, 9), A=st.sampled_from([1, 8, 32]), t0=st.integers(0, 50),
       seed=st.integers(0, 2 ** 32), skip_mask=st.integers(0, 511), gs=st.sampled_from([1.0, 0.5, 0.125, 3.0]),
       lr0=st.sampled_from([1e-3, 3e-4, 0.1]), mode=st.sampled_from([gi.GRAD_UNIFORM, gi.GRAD_LLM]),
       threads=st.sampled_from([1, 3]))
def test_host_replay_equals_oracle(n, K, A, t0, seed, skip_mask, gs, lr0, mode, threads):
    G = _G()
    if K > -(-n // A):
        return
    p0, m0, v0 = gi.warm_state(seed, n) if t0 else gi.cold_state(seed, n)
    recs, lrecs, t = [], [], t0
    for i in range(1, K + 1):
        skip = bool((skip_mask >> (i - 1)) & 1) and t > 0
        if not skip:
            t += 1
        lr = lr0 * (1 + 0.1 * i)
        recs.append(oracle.make_step_record(t=t, lr=lr, grad_scale=gs, skip=skip, **HP))
        lrecs.append(G.make_step_record(0.9, 0.999, 1e-8, 0.01, max(t, 1), lr, gs, skip))
    grads = [gi.grad_bits(seed, t0 + i, n, mode=mode) for i in range(1, K + 1)]
    parts = oracle.make_parts(n, K, A)
    cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, recs, parts)
    want = oracle.replay(cap, glog, recs, parts)
    o1 = oracle.trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]
    p, m, v = (np.ascontiguousarray(x) for x in oracle.assemble(cap))
    G.replay_host(lrecs, parts, p, m, v, [np.ascontiguousarray(g) for g in glog], threads=threads)
    for got, a, b in zip((p, m, v), want, o1):
        assert np.array_equal(got.view(np.uint32), a.view(np.uint32))
        assert np.array_equal(got.view(np.uint32), b.view(np.uint32))
