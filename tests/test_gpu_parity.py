"""GPU parity of the CUDA path against the oracle (-m gpu; calls go through the C ABI).

Bar (BASELINE.json north_star): pack and copy bit-exact; replayed fp32 state
bit-exact against the GPU's own synchronous snapshot; within 1e-6 max relative
error of the CPU oracle per element (expected: 0, the op order is pinned).
Sizes span many 2048-element tiles plus a ragged tail.
"""

import os

import numpy as np
import pytest
import torch

import gockpt_inputs as gi
import oracle
from gpu_helpers import HP, up_f32, up_u16, down_f32, down_u16, assert_state_equal, session_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2511_07035_b200 import build as gbuild
    gbuild.build()
    import paper_2511_07035_b200 as G
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device"
    assert G.device_count() >= 1
    return G


def _make_ctx(G, state, K, **kw):
    p, m, v = (up_f32(x) for x in state)
    out = torch.zeros(p.numel(), dtype=torch.int16, device="cuda")
    kw.setdefault("k_min", 1)
    kw.setdefault("k_max", max(K, 8))
    ctx = G.GoCkpt(p, m, v, out, **HP, **kw)
    return ctx, (p, m, v, out)


# ---------------------------------------------------------------- generator (harness) parity
@pytest.mark.parametrize("n,offset", [(1, 0), (1000, 17), (1 << 20, 5_000_000_007)])
def test_generator_matches_numpy(G, n, offset):
    for kind, mode, fn in [(1, 0, lambda: gi.master(42, n, offset)), (1, 1, lambda: gi.master(42, n, offset, 1)),
                           (2, 0, lambda: gi.exp_avg(42, n, offset)), (3, 0, lambda: gi.exp_avg_sq(42, n, offset))]:
        t = torch.empty(n, dtype=torch.float32, device="cuda")
        G.h_generate(kind, t, 42, 0, offset, mode)
        assert np.array_equal(down_f32(t).view(np.uint32), fn().view(np.uint32)), (kind, mode)
    for mode in (gi.GRAD_UNIFORM, gi.GRAD_LLM):
        t = torch.empty(n, dtype=torch.int16, device="cuda")
        G.h_generate(4, t, 7, 123, offset, mode, 4)
        assert np.array_equal(down_u16(t), gi.grad_bits(7, 123, n, offset, mode=mode, zero_per_256=4))


# ---------------------------------------------------------------- a2 without a session
@pytest.mark.parametrize("n", [1, 7, 8, 2048 * 37 + 5, 1_000_003])
def test_fused_step_trajectory_vs_oracle(G, n):
    seed, t0, steps = 11, 50, 4
    state, grads, recs, sargs = session_inputs(seed, n, steps, t0)
    p, m, v = (up_f32(x) for x in state)
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    want = oracle.trajectory(*state, grads, recs)
    for k in range(steps):
        r = G.make_step_record(HP["beta1"], HP["beta2"], HP["eps"], HP["weight_decay"], sargs[k]["adam_t"],
                               sargs[k]["lr"], sargs[k]["grad_scale"], sargs[k]["skip"])
        G.adamw_step(r, p, m, v, up_u16(grads[k]), out)
        torch.cuda.synchronize()
        assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), want[k + 1], f"step {k + 1}")
        assert np.array_equal(down_u16(out), oracle.rne_bf16(want[k + 1][0]))


# ---------------------------------------------------------------- the full session, staged + replays
@pytest.mark.parametrize("n,K,A,R,copy", [
    (1 << 20, 4, 1024, 2, "ce"),            # config 1
    (1_000_003, 4, 1024, 2, "ce"),          # ragged tail
    (1_000_003, 4, 1024, 1, "ce"),          # single slot
    (1 << 20, 4, 1024, 2, "zerocopy"),      # zero-copy drain
    (300_007, 8, 8, 2, "ce"),               # fine alignment, K=8
    (5000, 5, 8, 2, "zerocopy"),
    (64, 8, 8, 1, "ce"),                    # one unit per part
    (1 << 20, 1, 1024, 2, "ce"),            # K=1: a plain snapshot, no gradients
    (300_007, 64, 8, 2, "ce"),              # K = GCK_K_LIMIT (maximum), TMA kernel, parts not tile-aligned
])
@pytest.mark.parametrize("seed", [42, 7])
@pytest.mark.parametrize("plan", ["equal", "balanced"])
def test_session_staged_replays_and_snapshot(G, n, K, A, R, copy, seed, plan):
    t0 = 10
    state, grads, recs, sargs = session_inputs(seed, n, K, t0)
    ctx, (p, m, v, out) = _make_ctx(G, state, K, part_align=A, ring_slots=R, copy_mode=copy, eager_replay=False,
                                    chunk_bytes=(1 << 20) if copy == "ce" and R == 1 else 0, plan=plan)
    parts = (oracle.make_parts_balanced if plan == "balanced" else oracle.make_parts)(n, K, A)
    assert G.plan_parts(n, K, A, plan=plan) == parts
    g_dev = [up_u16(g) for g in grads]
    ctx.begin_checkpoint(t0, K)
    snap = None
    for i in range(1, K + 1):
        if i == K:
            snap = ctx.sync_snapshot()                   # S(T), T = t0+K-1: the reference
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], g_dev[i - 1], a["grad_scale"], a["skip"])
    torch.cuda.synchronize()
    # live state after update t0+K equals the oracle trajectory
    traj = oracle.trajectory(*state, grads, recs)
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), traj[K], "live S(t0+K)")
    assert_state_equal(snap, traj[K - 1], "sync snapshot S(T)")
    # staged bytes == the oracle's capture (pack + copy are bit copies, V4)
    ctx.wait_drained()
    st = ctx.staged()
    assert st["parts"] == parts and st["K"] == K and st["t0"] == t0
    cap, glog, _ = oracle.capture_session(*state, grads, recs, parts)
    assert_state_equal((st["master"], st["exp_avg"], st["exp_avg_sq"]), oracle.assemble(cap), "staged")
    assert len(st["glog"]) == K - 1
    for i in range(K - 1):
        assert np.array_equal(st["glog"][i], glog[i]), f"glog {i + 1}"
    # GPU replay (V6) == snapshot
    dP, dM, dV = (torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3))
    dG = torch.empty(max(1, n * (K - 1) + 128 * K), dtype=torch.int16, device="cuda")
    ctx.replay_gpu(dP, dM, dV, dG)
    assert_state_equal((down_f32(dP), down_f32(dM), down_f32(dV)), snap, "gpu replay vs snapshot")
    # host replay at finalize (V5) == snapshot == oracle O2 == oracle O1 (V7)
    ck = ctx.finalize()
    assert ck.step == t0 + K - 1
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), snap, "host replay vs snapshot")
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), oracle.replay(cap, glog, recs, parts), "vs O2")
    s = ctx.stats()
    assert s["sessions"] == 1 and s["session_steps"] == K
    assert s["d2h_bytes"] == oracle.session_bytes(parts)
    ctx.release()
    ctx.close()


def test_skipped_step_inside_session(G):
    n, K, t0 = 200_000, 4, 30
    state, grads, recs, sargs = session_inputs(3, n, K, t0, skips={t0 + 2})
    ctx, (p, m, v, out) = _make_ctx(G, state, K, part_align=64)
    ctx.begin_checkpoint(t0, K)
    g_dev = [up_u16(g) for g in grads]
    for i in range(1, K + 1):
        if i == K:
            snap = ctx.sync_snapshot()
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], g_dev[i - 1], a["grad_scale"], a["skip"])
    ck = ctx.finalize()
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), snap, "skip: host replay vs snapshot")
    want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, "skip: vs oracle")
    ctx.release()
    ctx.close()


# ---------------------------------------------------------------- eager replay, several sessions, plain steps
def test_eager_replay_multiple_sessions_with_plain_steps(G):
    n, K = 1 << 20, 4
    seed = 5
    state = gi.warm_state(seed, n)
    p, m, v = (up_f32(x) for x in state)
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=2, k_max=8, eager_replay=True)
    ref = tuple(x.copy() for x in state)
    step, t = 0, 0
    for sess in range(3):
        Ks = (K, 2, 8)[sess]
        for _ in range(3):                               # plain steps between sessions
            step += 1
            t += 1
            g = gi.grad_bits(seed, step, n)
            ctx.submit(0, step, t, 1e-3, up_u16(g))
            ref = oracle.adamw_update(*ref, g, oracle.make_step_record(t=t, lr=1e-3, **HP))[:3]
        ctx.begin_checkpoint(step, Ks)
        target = None
        for i in range(1, Ks + 1):
            step += 1
            t += 1
            g = gi.grad_bits(seed, step, n)
            ctx.submit(i, step, t, 1e-3, up_u16(g))
            ref = oracle.adamw_update(*ref, g, oracle.make_step_record(t=t, lr=1e-3, **HP))[:3]
            if i == Ks - 1 or Ks == 1:
                target = tuple(x.copy() for x in ref)
        # training continues while the checkpoint completes in the background
        step += 1
        t += 1
        g = gi.grad_bits(seed, step, n)
        ctx.submit(0, step, t, 1e-3, up_u16(g))
        ref = oracle.adamw_update(*ref, g, oracle.make_step_record(t=t, lr=1e-3, **HP))[:3]
        ck = None
        while ck is None:
            ck = ctx.finalize(block=False)
        assert ck.step == step - 2
        assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), target, f"session {sess}")
        ctx.release()
    torch.cuda.synchronize()
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), ref, "live")
    s = ctx.stats()
    assert s["sessions"] == 3 and s["stall_ms_total"] >= 0
    ctx.close()


# ---------------------------------------------------------------- torn read
def test_scribbled_live_state_does_not_reach_the_checkpoint(G):
    # SPEC torn-read freedom: the drain reads the slot, never live memory. Right after
    # the last session step's kernel, overwrite the live state on the compute stream; the
    # checkpoint must still be S(T).
    n, K, t0 = 1 << 20, 4, 10
    state, grads, recs, sargs = session_inputs(9, n, K, t0)
    ctx, (p, m, v, out) = _make_ctx(G, state, K, eager_replay=True)
    ctx.begin_checkpoint(t0, K)
    for i in range(1, K + 1):
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
        p.fill_(float("nan"))
        m.fill_(-7.0)
        v.fill_(123.0)
        # restore the true trajectory so the next step's capture is meaningful
        traj_i = oracle.trajectory(*state, grads[:i], recs[:i])[-1]
        p.copy_(up_f32(traj_i[0]))
        m.copy_(up_f32(traj_i[1]))
        v.copy_(up_f32(traj_i[2]))
    ck = ctx.finalize()
    want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, "scribbled")
    ctx.release()
    ctx.close()


# ---------------------------------------------------------------- protocol errors through the ABI
def test_protocol_errors(G):
    from paper_2511_07035_b200 import GckError
    from paper_2511_07035_b200 import _lib as L
    n, K, t0 = 4096, 4, 3
    state, grads, recs, sargs = session_inputs(1, n, K, t0)
    ctx, (p, m, v, out) = _make_ctx(G, state, K, part_align=8, k_min=2, k_max=4)
    g = up_u16(grads[0])

    def status_of(fn, *a):
        try:
            fn(*a)
        except GckError as e:
            return e.status
        return L.OK

    assert status_of(ctx.begin_checkpoint, t0, 5) == L.E_INVALID        # K > k_max
    assert status_of(ctx.begin_checkpoint, t0, 1) == L.E_INVALID        # K < k_min
    assert status_of(ctx.finalize) == L.E_PROTOCOL                      # no session
    assert status_of(ctx.release) == L.E_PROTOCOL
    assert status_of(ctx.submit, 1, t0 + 1, 1, 1e-3, g) == L.E_PROTOCOL  # session submit, no session
    ctx.begin_checkpoint(t0, K)
    assert status_of(ctx.begin_checkpoint, t0, K) == L.E_PROTOCOL       # begin twice
    assert status_of(ctx.submit, 0, t0 + 1, 1, 1e-3, g) == L.E_PROTOCOL  # plain submit inside a session
    assert status_of(ctx.submit, 2, t0 + 2, 1, 1e-3, g) == L.E_STALE     # skipped part 1
    assert status_of(ctx.submit, 1, t0 + 5, 1, 1e-3, g) == L.E_STALE     # step != t0 + part
    assert status_of(ctx.submit, 1, t0 + 1, 0, 1e-3, g) == L.E_INVALID   # adam_t = 0
    ctx.submit(1, t0 + 1, 1, 1e-3, g)
    assert status_of(ctx.finalize) == L.E_PROTOCOL                      # before part K
    for i in range(2, K + 1):
        ctx.submit(i, t0 + i, i, 1e-3, g)
    assert status_of(ctx.begin_checkpoint, t0 + K, K) == L.E_PROTOCOL   # unreleased checkpoint
    ck = ctx.finalize()
    assert ck.step == t0 + K - 1
    assert status_of(ctx.begin_checkpoint, t0 + K, K) == L.E_PROTOCOL
    ctx.release()
    ctx.begin_checkpoint(t0 + K, 2)                                       # next session is fine
    ctx.close()
    # misaligned gradient
    ctx2, _ = _make_ctx(G, state, K, part_align=8)
    gbuf = torch.zeros(n + 8, dtype=torch.int16, device="cuda")
    assert status_of(ctx2.submit, 0, 1, 1, 1e-3, gbuf[1:n + 1]) == L.E_INVALID
    ctx2.close()


# ---------------------------------------------------------------- a3 without a session
@pytest.mark.parametrize("nbytes", [16, 4096 + 16, (1 << 24) + 48])
@pytest.mark.parametrize("mode,chunk,ctas", [("ce", 0, 0), ("ce", 1 << 20, 0), ("zerocopy", 0, 7), ("zerocopy", 0, 148)])
def test_d2h_copy_byte_exact(G, nbytes, mode, chunk, ctas):
    src = torch.empty((nbytes + 1) // 2, dtype=torch.int16, device="cuda")
    G.h_generate(4, src, 99, 1, 0, 0, 0)
    dst = torch.zeros(nbytes + 64, dtype=torch.uint8, pin_memory=True)
    G.d2h_copy(dst, src, nbytes, mode, chunk, ctas)
    torch.cuda.synchronize()
    assert torch.equal(dst[:nbytes], src.view(torch.uint8)[:nbytes].cpu())
    assert not dst[nbytes:].any()          # nothing written past the end


# ---------------------------------------------------------------- NEXT-1: persist + crash + restore + resume
@pytest.mark.parametrize("replay_mode,k_max2", [("host", 4), ("deferred", 4), ("deferred", 2)])
def test_persist_restore_resume_equals_uninterrupted(G, tmp_path, replay_mode, k_max2):
    """SPEC S:506 recovery correctness: train, checkpoint (GoCkpt session), persist in the
    background, keep training, 'crash', restore from LATEST into a fresh context, resume at T+1
    with the same gradients -> bit-identical to the run that never crashed. replay_mode
    "deferred" (replay-on-restore, NEXT-2): the file carries the captured parts + gradient log and
    the restore replays on the GPU (k_max2 = 2 < K: the log does not fit the restoring context's
    arena and goes through a temporary buffer)."""
    from oracle import ckpt_file as OF
    n, K, seed = 300_007, 4, 21
    state = gi.warm_state(seed, n)
    total = 20
    grads = [gi.grad_bits(seed, s, n) for s in range(1, total + 1)]

    def train(ctx, steps, begin_at=None):
        for s in steps:
            part = 0
            if begin_at is not None and begin_at < s <= begin_at + K:
                if s == begin_at + 1:
                    ctx.begin_checkpoint(begin_at, K)
                part = s - begin_at
            ctx.submit(part, s, s, 1e-3, up_u16(grads[s - 1]))

    # uninterrupted reference run
    p, m, v = (up_f32(x) for x in state)
    ref = G.GoCkpt(p, m, v, None, **HP, k_min=K, k_max=K, part_align=64)
    train(ref, range(1, total + 1))
    torch.cuda.synchronize()
    want = (down_f32(p), down_f32(m), down_f32(v))
    ref.close()
    # run with a checkpoint over steps 6..9 (T = 8), persisted while training continues to 13
    p, m, v = (up_f32(x) for x in state)
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=K, k_max=K, part_align=64, replay_mode=replay_mode)
    train(ctx, range(1, 10), begin_at=5)
    ck = ctx.finalize()
    assert ck.step == 8 and ck.K == K and ck.replay_pending == (replay_mode == "deferred")
    path = str(tmp_path / "ckpt_8.rank0.bin")
    ctx.persist_begin(path, 0, 1, '{"note": "test"}')
    train(ctx, range(10, 14))
    st = ctx.persist_wait()
    assert st["bytes"] > 12 * n
    ctx.release()
    ctx.close()                                                   # the crash
    hdr, *s8 = OF.read_consistent(OF.latest(str(tmp_path)))      # the independent reader (+ oracle replay)
    assert hdr["step"] == 8 and hdr["adam_t"] == 8
    assert hdr.get("version", 1) == (2 if replay_mode == "deferred" else 1)
    recs8 = [oracle.make_step_record(t=s, lr=1e-3, **HP) for s in range(1, 9)]
    assert_state_equal(tuple(s8), oracle.trajectory(*state, grads[:8], recs8)[-1], "file vs oracle S(8)")
    # fresh process state: garbage tensors, restore, resume at T+1 = 9
    p2, m2, v2 = (torch.full((n,), 7.0, device="cuda") for _ in range(3))
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    ctx2 = G.GoCkpt(p2, m2, v2, out, **HP, k_min=1, k_max=k_max2, part_align=64)
    h = ctx2.restore(OF.latest(str(tmp_path)))
    assert h["step"] == 8
    torch.cuda.synchronize()
    assert_state_equal((down_f32(p2), down_f32(m2), down_f32(v2)), tuple(s8), "restored S(8)")
    assert np.array_equal(down_u16(out), oracle.rne_bf16(down_f32(p2)))   # working copy re-derived
    train(ctx2, range(h["step"] + 1, total + 1))
    torch.cuda.synchronize()
    assert_state_equal((down_f32(p2), down_f32(m2), down_f32(v2)), want, "resumed vs uninterrupted")
    ctx2.close()


# ---------------------------------------------------------------- NEXT-2: replay-on-restore
@pytest.mark.parametrize("n,K,A,staging", [(1 << 20, 4, 1024, "ring"), (1_000_003, 8, 1024, "ring"),
                                           (300_007, 3, 8, "direct"), (5000, 1, 8, "ring"),
                                           ((1 << 18) + 4101, 16, 1024, "ring")])
@pytest.mark.parametrize("plan", ["equal", "balanced"])
def test_deferred_replay_session_restore(G, tmp_path, n, K, A, staging, plan):
    """replay_mode="deferred": finalize leaves the captured parts (== the oracle's capture, bit for
    bit), persist writes them with the gradient log, and the GPU restore (replay kernel in place on
    the device tensors) and the host loader both give the oracle's S(T) bit for bit."""
    t0, seed = 10, 13
    state, grads, recs, sargs = session_inputs(seed, n, K, t0, skips=(t0 + 2,) if K >= 3 else ())
    ctx, (p, m, v, out) = _make_ctx(G, state, K, part_align=A, staging=staging, replay_mode="deferred", plan=plan)
    parts = (oracle.make_parts_balanced if plan == "balanced" else oracle.make_parts)(n, K, A)
    cap, glog, live = oracle.capture_session(*state, grads, recs, parts)
    want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
    ctx.begin_checkpoint(t0, K)
    gbuf = None
    for i in range(1, K + 1):
        a = sargs[i - 1]
        if staging == "direct":
            if gbuf is None:
                gbuf = up_u16(grads[i - 1])
            else:
                gbuf.copy_(up_u16(grads[i - 1]))
            ctx.submit(i, a["step"], a["adam_t"], a["lr"], gbuf, a["grad_scale"], a["skip"])
            ctx.grad_fence()
        else:
            ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
    ck = ctx.finalize()
    assert ck.step == t0 + K - 1 and ck.replay_pending == (K > 1)
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), oracle.assemble(cap), "captured parts")
    path = str(tmp_path / "d.bin")
    ctx.persist_begin(path)
    ctx.persist_wait()
    ctx.release()
    torch.cuda.synchronize()
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), live, "live S(t0+K)")
    hp_, hm_, hv_, hdr, _ = G.load_checkpoint(path, n, threads=4)            # host replay at load
    assert hdr["step"] == t0 + K - 1
    assert_state_equal((hp_, hm_, hv_), want, "host-loaded S(T)")
    h = ctx.restore(path)                                                   # GPU replay at restore
    torch.cuda.synchronize()
    assert h["step"] == t0 + K - 1
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), want, "GPU-restored S(T)")
    assert np.array_equal(down_u16(out), oracle.rne_bf16(want[0]))
    ctx.close()


# ---------------------------------------------------------------- a5 streaming host replay
@pytest.mark.parametrize("n,K,A,B,staging,copy", [(1 << 20, 4, 1024, 2, "ring", "ce"),
                                                  (1_000_003, 8, 1024, 2, "ring", "ce"),
                                                  (1_000_003, 8, 1024, 0, "ring", "ce"),     # default B (4)
                                                  (1_000_003, 8, 1024, 1, "ring", "zerocopy"),
                                                  (300_007, 6, 8, 3, "direct", "ce"),
                                                  (5000, 2, 8, 2, "ring", "ce"),
                                                  ((1 << 18) + 4101, 16, 1024, 4, "ring", "ce"),
                                                  (1 << 20, 1, 1024, 2, "ring", "ce")])
@pytest.mark.parametrize("plan", ["equal", "balanced"])
def test_streaming_replay_session(G, n, K, A, B, staging, copy, plan):
    """replay_mode="stream": slice i's update is applied to [0, hi_i) as soon as it drains, the
    gradient log is a ring of B buffers (the next drain into a buffer waits for its update).
    Result == the oracle's S(T) and == the GPU's own sync snapshot, bit for bit, with a skipped
    update inside the session."""
    t0, seed = 10, 19
    state, grads, recs, sargs = session_inputs(seed, n, K, t0, skips=(t0 + 2,) if K >= 3 else ())
    ctx, (p, m, v, out) = _make_ctx(G, state, K, part_align=A, staging=staging, copy_mode=copy,
                                    replay_mode="stream", stream_buffers=B, plan=plan)
    want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
    ctx.begin_checkpoint(t0, K)
    gbuf = None
    for i in range(1, K + 1):
        a = sargs[i - 1]
        if i == K:
            snap = ctx.sync_snapshot()
        if staging == "direct":
            if gbuf is None:
                gbuf = up_u16(grads[i - 1])
            else:
                gbuf.copy_(up_u16(grads[i - 1]))
            ctx.submit(i, a["step"], a["adam_t"], a["lr"], gbuf, a["grad_scale"], a["skip"])
            ctx.grad_fence()
        else:
            ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
    ck = ctx.finalize()
    assert ck.step == t0 + K - 1 and not ck.replay_pending
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), snap, "stream vs GPU sync snapshot")
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, "stream vs oracle")
    st = ctx.stats()
    assert st["last_stream_wait_ms"] >= 0 and st["last_session_k"] == K
    ctx.release()
    # a second session on the same context (buffers reused across sessions)
    t1 = t0 + K
    state2 = (down_f32(p), down_f32(m), down_f32(v))
    g2 = [gi.grad_bits(seed + 1, t1 + i, n) for i in range(1, K + 1)]
    ctx.begin_checkpoint(t1, K)
    for i in range(1, K + 1):
        gg = up_u16(g2[i - 1])
        if staging == "direct":
            gbuf.copy_(gg)
            gg = gbuf
        ctx.submit(i, t1 + i, sargs[-1]["adam_t"] + i, 1e-3, gg)
        if staging == "direct":
            ctx.grad_fence()
    ck = ctx.finalize()
    recs2 = [oracle.make_step_record(t=sargs[-1]["adam_t"] + i, lr=1e-3, **HP) for i in range(1, K + 1)]
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq),
                       oracle.trajectory(*state2, g2[:K - 1], recs2[:K - 1])[-1], "second session")
    with pytest.raises(Exception):
        ctx.staged()                                   # no staged view in streaming mode
    ctx.release()
    ctx.close()


# ---------------------------------------------------------------- NEXT-2: direct staging (GoCkpt-O literal)
@pytest.mark.parametrize("n,K,A,copy,staging", [(1 << 20, 4, 1024, "ce", "direct"), (1_000_003, 8, 1024, "ce", "direct"),
                                                (300_007, 3, 8, "zerocopy", "direct"), (1 << 20, 1, 1024, "ce", "direct"),
                                                (1_000_003, 4, 1024, "ce", "blocking")])
@pytest.mark.parametrize("plan", ["equal", "balanced"])
def test_direct_staging_session(G, n, K, A, copy, staging, plan):
    """No HBM ring: part i is copied from the live arrays during step t0+i's F/B, the gradient
    prefix from ONE reused gradient buffer that the 'backward' overwrites right after
    gck_grad_fence. Staged bytes, host replay, GPU replay and snapshot as in ring mode."""
    t0, seed = 10, 5
    state, grads, recs, sargs = session_inputs(seed, n, K, t0)
    p, m, v = (up_f32(x) for x in state)
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=1, k_max=max(K, 8), part_align=A, copy_mode=copy,
                   eager_replay=False, staging=staging, plan=plan)
    gbuf = torch.empty(n, dtype=torch.int16, device="cuda")
    for s in range(1, 3):                                   # plain steps before the session
        gbuf.copy_(up_u16(gi.grad_bits(seed, 1000 + s, n)))
        ctx.submit(0, t0 - 3 + s, t0 - 3 + s, 1e-3, gbuf)
    torch.cuda.synchronize()
    state = (down_f32(p), down_f32(m), down_f32(v))       # S(t0) after those steps
    ctx.begin_checkpoint(t0, K)
    snap = None
    for i in range(1, K + 1):
        ctx.grad_fence()                                    # the next backward may overwrite gbuf
        gbuf.copy_(up_u16(grads[i - 1]))
        if i == K:
            snap = ctx.sync_snapshot()
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], gbuf, a["grad_scale"], a["skip"])
    ctx.grad_fence()
    gbuf.fill_(0)                                          # scribble the gradient buffer afterwards
    ctx.wait_drained()
    parts = (oracle.make_parts_balanced if plan == "balanced" else oracle.make_parts)(n, K, A)
    cap, glog, _ = oracle.capture_session(*state, grads, recs, parts)
    st = ctx.staged()
    assert st["parts"] == parts
    assert_state_equal((st["master"], st["exp_avg"], st["exp_avg_sq"]), oracle.assemble(cap), "direct staged")
    for i in range(K - 1):
        assert np.array_equal(st["glog"][i], glog[i]), f"direct glog {i + 1}"
    dP, dM, dV = (torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3))
    dG = torch.empty(max(1, n * (K - 1) + 128 * K), dtype=torch.int16, device="cuda")
    ctx.replay_gpu(dP, dM, dV, dG)
    assert_state_equal((down_f32(dP), down_f32(dM), down_f32(dV)), snap, "direct gpu replay vs snapshot")
    ck = ctx.finalize()
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), snap, "direct host replay vs snapshot")
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), oracle.replay(cap, glog, recs, parts), "direct vs O2")
    assert ctx.stats()["d2h_bytes"] == oracle.session_bytes(parts)
    ctx.release()
    ctx.close()


# ---------------------------------------------------------------- the boundary from plain C
def test_c_api_demo_program(G, tmp_path, repo_root):
    """The ABI is usable from C without Python or torch: build examples/c_api_demo.c with gcc against
    include/gockpt.h + libgockpt.so, run a session, checkpoint == synchronous snapshot."""
    import subprocess
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    exe = str(tmp_path / "c_api_demo")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(repo_root, "include"), "-I", os.path.join(cuda, "include"),
                    os.path.join(repo_root, "examples", "c_api_demo.c"), "-L", os.path.dirname(G.LIB_PATH),
                    "-l:libgockpt.so", "-L", os.path.join(cuda, "lib64"), "-lcudart",
                    f"-Wl,-rpath,{os.path.dirname(G.LIB_PATH)}", "-o", exe], check=True)
    for n, K in [((1 << 20) + 7, 4), (124_439_808, 8)]:
        r = subprocess.run([exe, str(n), str(K)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "== the synchronous snapshot" in r.stdout, r.stdout + r.stderr


# ---------------------------------------------------------------- failure path: checkpoint aborted, training continues
@pytest.mark.parametrize("staging,replay_mode", [("ring", "host"), ("direct", "host"), ("ring", "stream"),
                                                 ("direct", "stream")])
def test_drain_failure_aborts_checkpoint_not_training(G, staging, replay_mode):
    """a transfer-channel failure aborts the checkpoint (finalize reports it)
    while every optimizer update still runs; the next session works normally."""
    from paper_2511_07035_b200 import GckError
    from paper_2511_07035_b200 import _lib as L
    n, K, t0, seed = 300_007, 4, 10, 13
    state, grads, recs, sargs = session_inputs(seed, n, 2 * K, t0)
    p, m, v = (up_f32(x) for x in state)
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=K, k_max=K, part_align=64, staging=staging, replay_mode=replay_mode,
                   stream_buffers=1)
    os.environ["GCK_FAULT_DRAIN"] = "2"
    try:
        ctx.begin_checkpoint(t0, K)
        statuses = []
        for i in range(1, K + 1):
            a = sargs[i - 1]
            try:
                ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
                statuses.append(L.OK)
            except GckError as e:
                statuses.append(e.status)
    finally:
        os.environ.pop("GCK_FAULT_DRAIN", None)
    assert statuses[0] == L.OK and all(s_ == L.E_ABORTED for s_ in statuses[1:]), statuses
    with pytest.raises(GckError) as e:
        ctx.finalize()
    assert e.value.status == L.E_ABORTED
    torch.cuda.synchronize()
    traj = oracle.trajectory(*state, grads, recs)
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), traj[K], "training continued through the abort")
    # the next session (steps t0+K+1 .. t0+2K) checkpoints normally
    ctx.begin_checkpoint(t0 + K, K)
    for i in range(1, K + 1):
        a = sargs[K + i - 1]
        if i == K:
            snap = ctx.sync_snapshot()
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[K + i - 1]), a["grad_scale"], a["skip"])
    ck = ctx.finalize()
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), snap, "session after the abort")
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), traj[2 * K - 1], "session after the abort vs oracle")
    ctx.release()
    ctx.close()


@pytest.mark.parametrize("numa", [0, -1, -2])
def test_numa_bound_arena_session(G, numa):
    """The pinned arena from mmap + mbind + cudaHostRegister on an explicit node (0), the GPU's own
    node (-1; unbound when the platform reports none), or cudaHostAlloc (-2): same bytes out."""
    n, K, t0 = 1 << 20, 4, 10
    state, grads, recs, sargs = session_inputs(17, n, K, t0)
    ctx, (p, m, v, out) = _make_ctx(G, state, K, numa_node=numa)
    ctx.begin_checkpoint(t0, K)
    for i in range(1, K + 1):
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
    ck = ctx.finalize()
    want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, f"numa {numa}")
    st = ctx.stats()
    if numa == 0:
        assert st["numa_node"] == 0
    if numa == -2:
        assert st["numa_node"] == -1
    ctx.release()
    ctx.close()


@pytest.mark.parametrize("n,K,staging,eager", [(1_000_003, 4, "ring", True), (1 << 20, 8, "direct", False),
                                              (124_439_808, 8, "ring", True)])
def test_gpu_replay_finalize_mode(G, n, K, staging, eager):
    """replay_mode='gpu': the consistency update runs in the replay kernel (stale parts and the
    gradient log uploaded to library scratch, consistent parts downloaded) — same bytes as the
    host replay and the synchronous snapshot."""
    t0, seed = 20, 8
    dev = torch.device("cuda", 0)
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m, v = torch.empty_like(p), torch.empty_like(p)
    G.h_generate(1, p, seed, 0, 0, 0)
    G.h_generate(2, m, seed)
    G.h_generate(3, v, seed)
    g = torch.empty(n, dtype=torch.int16, device=dev)
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=K, k_max=K, staging=staging, eager_replay=eager, replay_mode="gpu")
    ctx.begin_checkpoint(t0, K)
    for i in range(1, K + 1):
        ctx.grad_fence()
        G.h_generate(4, g, seed, t0 + i, 0, 1, 4)
        if i == K:
            snap = ctx.sync_snapshot()
        ctx.submit(i, t0 + i, t0 + i, 1e-3, g)
    ck = ctx.finalize()
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), snap, "gpu-replay finalize vs snapshot")
    assert ctx.stats()["replay_threads"] == 0
    ctx.release()
    ctx.close()


def test_caller_owned_ring(G):
    """SURVEY §8(b) ownership: PyTorch may own the HBM ring (caching-allocator accounting)."""
    from paper_2511_07035_b200 import GckError
    from paper_2511_07035_b200 import _lib as L
    n, K, t0 = 1_000_003, 4, 10
    state, grads, recs, sargs = session_inputs(23, n, K, t0)
    need = G.ring_bytes_required(n, K, K, 1024, 2)
    p, m, v = (up_f32(x) for x in state)
    with pytest.raises(GckError) as e:
        G.GoCkpt(p, m, v, None, **HP, k_min=K, k_max=K, ring=torch.empty(need - 256, dtype=torch.uint8, device="cuda"))
    assert e.value.status == L.E_INVALID
    ring = torch.empty(need, dtype=torch.uint8, device="cuda")
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=K, k_max=K, ring=ring)
    ctx.begin_checkpoint(t0, K)
    for i in range(1, K + 1):
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
    ck = ctx.finalize()
    want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, "caller-owned ring")
    ctx.release()
    ctx.close()
    del ring                                   # freed by torch, not by the library


@pytest.mark.parametrize("skip_at", [1, 3, 4])
def test_skip_positions(G, skip_at):
    n, K, t0 = 100_000, 4, 40
    state, grads, recs, sargs = session_inputs(29, n, K, t0, skips={t0 + skip_at})
    ctx, (p, m, v, out) = _make_ctx(G, state, K, part_align=64)
    ctx.begin_checkpoint(t0, K)
    for i in range(1, K + 1):
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
    ck = ctx.finalize()
    want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, f"skip at {skip_at}")
    torch.cuda.synchronize()
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), oracle.trajectory(*state, grads, recs)[-1], "live")
    ctx.release()
    ctx.close()


def test_two_contexts_interleaved_and_destroy_mid_session(G):
    """Two shards in one process with interleaved sessions (independent streams/events/arenas), and a
    context destroyed in the middle of a session (no leak of queued work into the survivor)."""
    n, K, t0 = 200_003, 4, 10
    sa = session_inputs(31, n, K, t0)
    sb = session_inputs(37, n, K, t0)
    ca, _ = _make_ctx(G, sa[0], K, part_align=64)
    cb, _ = _make_ctx(G, sb[0], K, part_align=64, staging="direct")
    cc, _ = _make_ctx(G, sa[0], K, part_align=64)
    for c in (ca, cb, cc):
        c.begin_checkpoint(t0, K)
    for i in range(1, K + 1):
        for c, (state, grads, recs, sargs) in ((ca, sa), (cb, sb), (cc, sa)):
            if c is cc and i >= 3:
                continue
            a = sargs[i - 1]
            c.grad_fence()
            c.submit(i, a["step"], a["adam_t"], a["lr"], up_u16(grads[i - 1]), a["grad_scale"], a["skip"])
        if i == 2:
            cc.close()                      # destroyed mid-session
    for c, (state, grads, recs, sargs) in ((ca, sa), (cb, sb)):
        ck = c.finalize()
        want = oracle.trajectory(*state, grads[:K - 1], recs[:K - 1])[-1]
        assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, "interleaved")
        c.release()
        c.close()


def test_automatic_k(G):
    """NEXT-4: begin_checkpoint(t0, 0) picks K from the measured step time and link rate; the
    session it runs is exact whatever K it picked."""
    n, t0, seed = 1 << 20, 30, 41
    state = gi.warm_state(seed, n)
    p, m, v = (up_f32(x) for x in state)
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=1, k_max=16, part_align=1024)
    ref = tuple(x.copy() for x in state)
    a = torch.randn(4096, 4096, device="cuda")
    for s in range(1, t0 + 1):                          # plain steps with some work between them
        torch.mm(a, a)
        g = gi.grad_bits(seed, s, n)
        ctx.submit(0, s, s, 1e-3, up_u16(g))
        ref = oracle.adamw_update(*ref, g, oracle.make_step_record(t=s, lr=1e-3, **HP))[:3]
    torch.cuda.synchronize()
    ctx.begin_checkpoint(t0, 0)
    st = ctx.stats()
    K = st["last_session_k"]
    assert 1 <= K <= 16 and st["auto_step_ms"] > 0
    target = None
    for i in range(1, K + 1):
        s = t0 + i
        g = gi.grad_bits(seed, s, n)
        ctx.submit(i, s, s, 1e-3, up_u16(g))
        ref = oracle.adamw_update(*ref, g, oracle.make_step_record(t=s, lr=1e-3, **HP))[:3]
        if i == K - 1 or K == 1:
            target = tuple(x.copy() for x in ref) if K > 1 else target
    ck = ctx.finalize()
    if K == 1:
        target = oracle.trajectory(*state, [gi.grad_bits(seed, s, n) for s in range(1, t0 + 1)],
                                   [oracle.make_step_record(t=s, lr=1e-3, **HP) for s in range(1, t0 + 1)])[-1]
    assert ck.step == t0 + K - 1
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), target, f"auto K={K}")
    ctx.release()
    ctx.close()


@pytest.mark.parametrize("replay_mode", ["host", "deferred"])
def test_checkpointed_adamw_training_loop(G, tmp_path, replay_mode):
    """The optimizer face (save_checkpoint / step / wait): checkpoints requested every 12 steps
    while training runs, each consistent == the oracle's state at its step and durable on disk.
    deferred (replay-on-restore): the handles hold the captured parts, the files S(T) after the
    oracle's replay, and opt.restore() brings the device state back to S(39) through the GPU replay."""
    from paper_2511_07035_b200.optim import CheckpointedAdamW
    from oracle import ckpt_file as OF
    n, K, seed, steps = 300_007, 4, 51, 40
    state = gi.warm_state(seed, n)
    p, m, v = (up_f32(x) for x in state)
    got = {}
    opt = CheckpointedAdamW(p, m, v, None, lr=1e-3, K=K, part_align=64, persist_dir=str(tmp_path),
                            replay_mode=replay_mode,
                            on_checkpoint=lambda ck: got.__setitem__(ck.step, (ck.master.copy(), ck.exp_avg.copy(),
                                                                               ck.exp_avg_sq.copy())))
    ref, traj = tuple(x.copy() for x in state), {0: tuple(x.copy() for x in state)}
    gbuf = torch.empty(n, dtype=torch.int16, device="cuda")
    for s in range(1, steps + 1):
        if s % 12 == 1:
            opt.save_checkpoint()
        opt.grad_fence()
        g = gi.grad_bits(seed, s, n)
        gbuf.copy_(up_u16(g))
        opt.step(gbuf)
        ref = oracle.adamw_update(*ref, g, oracle.make_step_record(t=s, lr=1e-3, **HP))[:3]
        traj[s] = tuple(x.copy() for x in ref)
    last = opt.wait()
    assert sorted(got) == [K - 1 + 12 * k for k in range(4)] == [3, 15, 27, 39]
    if replay_mode == "host":
        for step, st in got.items():
            assert_state_equal(st, traj[step], f"checkpoint at {step}")
    assert last[0] == 39 and OF.latest(str(tmp_path)) == last[1]
    hdr, fp, fm, fv = OF.read_consistent(last[1])
    assert hdr["step"] == 39 and hdr["adam_t"] == 39
    assert_state_equal((fp, fm, fv), traj[39], "persisted")
    h = opt.restore()                                        # device state back to S(39)
    torch.cuda.synchronize()
    assert h["step"] == 39 and opt.global_step == 39 and opt.adam_t == 39
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), traj[39], "restored")
    opt.close()


# ---------------------------------------------------------------- T2 on one GPU: R shards, R contexts
@pytest.mark.parametrize("n_total,R,K", [(1_200_007, 4, 4), (300_007, 3, 8)])   # TMA kernel (n_r >= 2^18); grid-stride kernel
def test_multi_shard_emulation_concatenates_to_global(G, n_total, R, K):
    """SURVEY §4.2 T2 "single-process multi-shard emulation on one GPU": R contexts over the R ZeRO-1
    shards of one flat vector (§4.5: every rank saves its own optimizer shard), each driven
    through the full GPU path (fused kernel + ring + drain + eager host replay) in lock-step from the
    same global step; the concatenated checkpoints equal the oracle's S(T) of the whole vector."""
    from paper_2511_07035_b200.harness import zero1_shard
    t0 = 10
    _, n_r, padded = zero1_shard(n_total, R, 0, align=1024)
    ctxs, grads = [], []
    for r in range(R):
        idx = np.arange(r * n_r, (r + 1) * n_r, dtype=np.uint64)
        ctx, _ = _make_ctx(G, gi.warm_state(42, idx), K, part_align=1024, eager_replay=True)
        ctxs.append(ctx)
        grads.append([up_u16(gi.grad_bits(42, t0 + i, idx)) for i in range(1, K + 1)])
    for ctx in ctxs:
        ctx.begin_checkpoint(t0, K)
    for i in range(1, K + 1):                      # one global step = every rank's update t0+i
        for r, ctx in enumerate(ctxs):
            ctx.submit(i, t0 + i, t0 + i, 1e-3, grads[r][i - 1])
    cks = [ctx.finalize() for ctx in ctxs]
    assert all(ck.step == t0 + K - 1 for ck in cks)
    got = [np.concatenate([getattr(ck, f) for ck in cks]) for f in ("master", "exp_avg", "exp_avg_sq")]
    idx = np.arange(padded, dtype=np.uint64)
    p0, m0, v0 = gi.warm_state(42, idx)
    recs = [oracle.make_step_record(t=t0 + i, lr=1e-3, **HP) for i in range(1, K)]
    want = oracle.trajectory(p0, m0, v0, [gi.grad_bits(42, t0 + i, idx) for i in range(1, K)], recs)[-1]
    assert_state_equal(got, want, f"{R} shards concatenated vs oracle S(T)")
    for ctx in ctxs:
        ctx.release()
        ctx.close()


# ---------------------------------------------------------------- a5 GPU replay kernel, any partition
@pytest.mark.parametrize("n,K,A,skip_at", [(1000, 2, 1, None), (5003, 5, 3, 2), (100_003, 9, 1, None),
                                           (300_007, 17, 8, 5), (2_000_003, 8, 1024, None), (65, 64, 1, 7)])
def test_replay_device_any_partition_vs_oracle(G, n, K, A, skip_at):
    """gck_replay_device (the part-interleaved replay kernel) on partitions whose boundaries are not
    8-element aligned (A = 1, 3), up to K = 64 parts, with a skipped update: the replayed state equals
    the oracle's O2 replay (and so S(T), O1) bit for bit."""
    t0, seed = 10, 3
    p0, m0, v0 = gi.warm_state(seed, n)
    grads = [gi.grad_bits(seed, t0 + i, n) for i in range(1, K + 1)]
    orecs, lrecs, t = [], [], t0
    for i in range(1, K + 1):
        sk = (i == skip_at)
        t += 0 if sk else 1
        orecs.append(oracle.make_step_record(t=max(t, 1), lr=1e-3, skip=sk, **HP))
        lrecs.append(G.make_step_record(HP["beta1"], HP["beta2"], HP["eps"], HP["weight_decay"], max(t, 1), 1e-3,
                                        skip=sk))
    parts = oracle.make_parts(n, K, A)
    assert G.plan_parts(n, K, A) == parts
    cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, orecs, parts)
    want = oracle.replay(cap, glog, orecs, parts)
    dp, dm, dv = (up_f32(np.ascontiguousarray(x)) for x in oracle.assemble(cap))
    dg = [up_u16(np.ascontiguousarray(g)) for g in glog]
    G.replay_device(lrecs, parts, dp, dm, dv, dg)
    torch.cuda.synchronize()
    assert_state_equal((down_f32(dp), down_f32(dm), down_f32(dv)), want, "GPU replay vs oracle O2")
    traj = oracle.trajectory(p0, m0, v0, grads[:K - 1], orecs[:K - 1])
    assert_state_equal((down_f32(dp), down_f32(dm), down_f32(dv)), traj[-1], "GPU replay vs oracle O1")
