"""GPU negative controls of the checkpoint path (-m gpu; SURVEY §8(c) V8, §8(b) error conventions).

A session whose slice never drained (GCK_FAULT_DROP_SLICE) must not be replayed around: finalize
reports GCK_E_INCOMPLETE and discards the checkpoint. A landed byte that differs from the
staged bytes (GCK_FAULT_FLIP) is caught by the drain verification (device checksum of the staged
sections vs host checksum of the landed ones) and finalize reports GCK_E_CORRUPT; with the
verification off, the same flip makes the checkpoint differ from the synchronous snapshot S(T).
Either way training continues bit-exactly (the oracle trajectory) and the next session checkpoints
normally.
"""

import os

import numpy as np
import pytest
import torch

import oracle
from gpu_helpers import HP, up_f32, up_u16, down_f32, assert_state_equal, session_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2511_07035_b200 import build as gbuild
    gbuild.build()
    import paper_2511_07035_b200 as G
    assert torch.cuda.is_available()
    return G


def _run(G, monkeypatch, hook, step, staging, replay_mode, verify=True, n=300_007, K=4):
    from paper_2511_07035_b200 import GckError
    t0, seed = 20, 17
    state, grads, recs, sargs = session_inputs(seed, n, 2 * K, t0)
    p, m, v = (up_f32(x) for x in state)
    ctx = G.GoCkpt(p, m, v, None, **HP, k_min=K, k_max=K, part_align=64, staging=staging, replay_mode=replay_mode,
                   verify_drain=verify)
    g_dev = [up_u16(g) for g in grads]
    monkeypatch.setenv(hook, str(step))
    ctx.begin_checkpoint(t0, K)
    monkeypatch.delenv(hook)
    snap = None
    for i in range(1, K + 1):
        a = sargs[i - 1]
        if i == K:
            snap = ctx.sync_snapshot()
        try:
            ctx.submit(i, a["step"], a["adam_t"], a["lr"], g_dev[i - 1], a["grad_scale"], a["skip"])
        except GckError as e:  # a streaming worker that already stopped voids the remaining steps
            assert replay_mode == "stream" and e.status == 7  # GCK_E_ABORTED
        if staging != "ring":
            ctx.grad_fence()
    status, ck = 0, None
    try:
        ck = ctx.finalize()
    except GckError as e:
        status = e.status
    torch.cuda.synchronize()
    traj = oracle.trajectory(*state, grads, recs)
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), traj[K], "training continued")
    # a normal session right after (steps t0+K+1 .. t0+2K)
    if ck is not None:
        ck = (ck.master.copy(), ck.exp_avg.copy(), ck.exp_avg_sq.copy())
    ctx.release()
    ctx.begin_checkpoint(t0 + K, K)
    for i in range(1, K + 1):
        a = sargs[K + i - 1]
        if i == K:
            snap2 = ctx.sync_snapshot()
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], g_dev[K + i - 1], a["grad_scale"], a["skip"])
        if staging != "ring":
            ctx.grad_fence()
    ck2 = ctx.finalize()
    if replay_mode == "deferred":  # the handle holds the captured parts; S(T) materialises at load
        assert ck2.replay_pending
    else:
        assert_state_equal((ck2.master, ck2.exp_avg, ck2.exp_avg_sq), snap2, "next session")
        assert_state_equal((ck2.master, ck2.exp_avg, ck2.exp_avg_sq), traj[2 * K - 1], "next session vs oracle")
    ctx.release()
    ctx.close()
    return status, ck, snap


@pytest.mark.parametrize("staging", ["ring", "direct"])
@pytest.mark.parametrize("replay_mode", ["host", "stream", "gpu"])
@pytest.mark.parametrize("step", [1, 3, 4])
def test_dropped_slice_is_incomplete(G, monkeypatch, staging, replay_mode, step):
    from paper_2511_07035_b200 import _lib as L
    status, ck, _ = _run(G, monkeypatch, "GCK_FAULT_DROP_SLICE", step, staging, replay_mode)
    assert status == L.E_INCOMPLETE and ck is None


@pytest.mark.parametrize("staging", ["ring", "direct"])
@pytest.mark.parametrize("replay_mode", ["host", "stream", "deferred"])
@pytest.mark.parametrize("step", [1, 4])
def test_flipped_byte_is_detected(G, monkeypatch, staging, replay_mode, step):
    from paper_2511_07035_b200 import _lib as L
    status, ck, _ = _run(G, monkeypatch, "GCK_FAULT_FLIP", step, staging, replay_mode)
    assert status == L.E_CORRUPT and ck is None


@pytest.mark.parametrize("step", [1, 4])
def test_flipped_byte_without_verification_differs_from_snapshot(G, monkeypatch, step):
    status, ck, snap = _run(G, monkeypatch, "GCK_FAULT_FLIP", step, "ring", "host", verify=False)
    assert status == 0
    differs = [not np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(ck, snap)]
    assert differs[0], "the corrupted master byte must show in the checkpoint"


@pytest.mark.parametrize("hook,status", [("GCK_FAULT_DRAIN", "GCK_E_ABORTED"), ("GCK_FAULT_DROP_SLICE", "GCK_E_INCOMPLETE"),
                                         ("GCK_FAULT_FLIP", "GCK_E_CORRUPT")])
def test_checkpointed_adamw_survives_a_voided_checkpoint(G, tmp_path, monkeypatch, hook, status):
    """The optimizer face through a failed checkpoint: the failure is recorded, the
    training trajectory is unaffected (== oracle), the next requested checkpoint is consistent and
    durable, and retention keeps only the 2 newest files on disk."""
    import gockpt_inputs as gi
    from oracle import ckpt_file as OF
    from paper_2511_07035_b200.optim import CheckpointedAdamW
    n, K, seed, steps = 300_007, 4, 23, 52
    state = gi.warm_state(seed, n)
    p, m, v = (up_f32(x) for x in state)
    opt = CheckpointedAdamW(p, m, v, None, lr=1e-3, K=K, part_align=64, persist_dir=str(tmp_path), keep=2)
    ref, traj = tuple(x.copy() for x in state), {}
    gbuf = torch.empty(n, dtype=torch.int16, device="cuda")
    for s in range(1, steps + 1):
        if s % 12 == 1:
            if s == 13:
                monkeypatch.setenv(hook, "2")   # the session of steps 13..16 (T = 15) fails at its step 2
            opt.save_checkpoint()
        g = gi.grad_bits(seed, s, n)
        gbuf.copy_(up_u16(g))
        opt.step(gbuf)
        if s == 14:  # GCK_FAULT_DRAIN is read at the drain (step 14); the others at begin (step 13)
            monkeypatch.delenv(hook)
        ref = oracle.adamw_update(*ref, g, oracle.make_step_record(t=s, lr=1e-3, **HP))[:3]
        traj[s] = tuple(x.copy() for x in ref)
    last = opt.wait()
    torch.cuda.synchronize()
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), traj[steps], "training through the failure")
    assert [f[:2] for f in opt.failures] == [(15, status)]
    assert last[0] == 51 and OF.latest(str(tmp_path)) == last[1]
    hdr, fp, fm, fv = OF.read_consistent(last[1])
    assert_state_equal((fp, fm, fv), traj[51], "persisted after the failure")
    files = sorted(f for f in os.listdir(tmp_path) if f.endswith(".bin"))
    assert files == ["ckpt_39.rank0.bin", "ckpt_51.rank0.bin"], files
    opt.close()
