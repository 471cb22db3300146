"""The n > 2^32 size class on one B200 (-m gpu): element indices past 2^32 through the fused kernel,
the ring, the drain, the host replay, the drain verification and the replay kernel.

SURVEY §8 sizes table: Llama-2 13B at 2 ranks is a 6.5G-element shard per rank (§4.5: each
rank saves its own optimizer shard), the only configuration with n > 2^32. A replayed part reaches
past 2^32 only if hi_{K-1} = n(K-1)/K > 2^32, so the session runs at n = 5e9 + 4101 (ragged) with
K = 8 (the last stale part ends near 4.375e9): 96 GB of HBM (state, gradient, bf16 params, one ring
slot) and 19n = 95 GB of pinned host memory plus the 60 GB synchronous snapshot.

Checks: the whole checkpoint == the GPU's own synchronous snapshot S(T) bit for bit; 16 windows
of 2^20 elements (every part boundary, both sides of 2^32, seeded random offsets, the tail) ==
the CPU oracle's S(T) computed on exactly those indices (the update is elementwise, so windows are
exact).
"""

import numpy as np
import pytest
import torch

import gockpt_inputs as gi
import oracle
from gpu_helpers import HP, assert_state_equal

pytestmark = pytest.mark.gpu

GEN_MASTER, GEN_M, GEN_V, GEN_GRAD = 1, 2, 3, 4


@pytest.fixture(scope="module")
def G():
    from paper_2511_07035_b200 import build as gbuild
    gbuild.build()
    import paper_2511_07035_b200 as G
    assert torch.cuda.is_available()
    return G


def _windows(n, parts, rng, w=1 << 20):
    starts = [0, n - w, (1 << 32) - w // 2, (1 << 32) + 12345]
    starts += [lo - w // 2 for lo, _ in parts[1:]]
    starts += list(rng.integers(0, n - w, 16 - len(starts)))
    out = []
    for s in starts:
        s = int(min(max(0, s), n - w))
        out.append(np.arange(s, s + w, dtype=np.uint64))
    return out


def _views(ck):
    return [np.asarray(x).view(np.uint32) for x in ck]


def test_session_past_2_32(G):
    n, K, t0, seed = 5_000_000_000 + 4101, 8, 30, 77
    lr = 1e-3
    dev = torch.device("cuda")
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m, v = torch.empty_like(p), torch.empty_like(p)
    G.h_generate(GEN_MASTER, p, seed, 0, 0, 0)
    G.h_generate(GEN_M, m, seed, 0, 0)
    G.h_generate(GEN_V, v, seed, 0, 0)
    out = torch.empty(n, dtype=torch.int16, device=dev)
    g = torch.empty(n, dtype=torch.int16, device=dev)
    ctx = G.GoCkpt(p, m, v, out, **HP, k_min=K, k_max=K, part_align=1024, ring_slots=1, eager_replay=True)
    parts = G.plan_parts(n, K, 1024)
    assert parts[K - 2][1] > (1 << 32), "a replayed part must reach past 2^32"
    ctx.begin_checkpoint(t0, K)
    snap = None
    for i in range(1, K + 1):
        G.h_generate(GEN_GRAD, g, seed, t0 + i, 0, gi.GRAD_LLM, 4)
        if i == K:
            snap = ctx.sync_snapshot()   # S(T), T = t0+K-1
        ctx.submit(i, t0 + i, t0 + i, lr, g)
    ck = ctx.finalize()
    assert ck.step == t0 + K - 1
    for name, a, b in zip(("master", "exp_avg", "exp_avg_sq"), _views((ck.master, ck.exp_avg, ck.exp_avg_sq)),
                          _views(snap)):
        assert np.array_equal(a, b), f"{name}: checkpoint != synchronous snapshot"
    del snap
    s = ctx.stats()
    assert s["d2h_bytes"] == oracle.session_bytes(parts)
    # oracle S(T) on windows
    recs = [oracle.make_step_record(t=t0 + i, lr=lr, **HP) for i in range(1, K)]
    for idx in _windows(n, parts, np.random.default_rng(seed)):
        st = gi.warm_state(seed, idx)
        grads = [gi.grad_bits(seed, t0 + i, idx, mode=gi.GRAD_LLM, zero_per_256=4) for i in range(1, K)]
        want = oracle.trajectory(*st, grads, recs)[-1]
        lo, hi = int(idx[0]), int(idx[-1]) + 1
        assert_state_equal((ck.master[lo:hi], ck.exp_avg[lo:hi], ck.exp_avg_sq[lo:hi]), want, f"window @{lo}")
    ctx.release()
    ctx.close()


def test_replay_kernel_past_2_32(G):
    """replay_kernel with a stale part ending past 2^32: one pending update over [0, 4.35e9) equals
    the fused kernel's update of the same elements (compared as bit patterns, on the device)."""
    n, cut, seed, t = 4_400_000_000, 4_350_001_152, 91, 57
    dev = torch.device("cuda")
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m, v = torch.empty_like(p), torch.empty_like(p)
    G.h_generate(GEN_MASTER, p, seed, 0, 0, 0)
    G.h_generate(GEN_M, m, seed, 0, 0)
    G.h_generate(GEN_V, v, seed, 0, 0)
    g = torch.empty(cut, dtype=torch.int16, device=dev)
    G.h_generate(GEN_GRAD, g, seed, t, 0, gi.GRAD_LLM, 4)
    rec = G.make_step_record(HP["beta1"], HP["beta2"], HP["eps"], HP["weight_decay"], t, 1e-3)
    ref = [x[:cut].clone() for x in (p, m, v)]
    G.adamw_step(rec, *ref, g)
    G.replay_device([rec, rec], [(0, cut), (cut, n)], p, m, v, [g])
    torch.cuda.synchronize()
    for a, b, name in zip((p, m, v), ref, ("master", "exp_avg", "exp_avg_sq")):
        assert torch.equal(a[:cut].view(torch.int32), b.view(torch.int32)), name
    # and one window past 2^32 against the CPU oracle
    idx = np.arange((1 << 32) + 1000, (1 << 32) + 1000 + (1 << 20), dtype=np.uint64)
    want = oracle.adamw_update(*gi.warm_state(seed, idx), gi.grad_bits(seed, t, idx, mode=gi.GRAD_LLM,
                                                                        zero_per_256=4),
                               oracle.make_step_record(t=t, lr=1e-3, **HP))[:3]
    lo, hi = int(idx[0]), int(idx[-1]) + 1
    got = tuple(x[lo:hi].cpu().numpy() for x in (p, m, v))
    assert_state_equal(got, want, "replay window past 2^32")
