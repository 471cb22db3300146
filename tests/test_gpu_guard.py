"""GPU parity through the fast-path guard's fallback branch (-m gpu; calls go through the C ABI).

The hot kernels (the TMA fused kernel's groups of 4, the replay kernel's groups of 8) compute the
normative update through branch-free division / sqrt
sequences and fall back to the IEEE intrinsics for the whole group when some lane's m' or v'
leaves the guarded ranges (|m'| in [2^-40, 2^20], |v'| in [2^-60, 2^60], adamw_math.cuh). The warm
synthetic states of the other GPU tests never leave them; here real training's cases do:

  - a cold start (S(0): m = v = 0) with the "llm" gradient's exact zeros (embedding
    rows absent from the batch): m' = v' = 0 at update 1, tiny moments after it;
  - planted lanes on single lanes of a group: m in {0, denormal, +-2^-45, +-2^25}, v in {0,
    denormal} with a zero gradient, and a step with grad_scale 2^20 (loss-scale unscaling).

Each session is checked against the oracle bit for bit (live state, staged bytes, GPU replay,
host replay), and each test asserts — from the oracle's own trajectory — that the guard failed
for some element update, so the fallback branch really ran on the device.
"""

import numpy as np
import pytest
import torch

import gockpt_inputs as gi
import oracle
from gpu_helpers import HP, up_f32, up_u16, down_f32, assert_state_equal

pytestmark = pytest.mark.gpu

# the kernels' guard ranges (adamw_math.cuh kG2Lo/kG3Hi, kG1Lo/kG1Hi); test bookkeeping only
M_LO, M_HI, V_LO, V_HI = 2.0 ** -40, 2.0 ** 20, 2.0 ** -60, 2.0 ** 60


@pytest.fixture(scope="module")
def G():
    from paper_2511_07035_b200 import build as gbuild
    gbuild.build()
    import paper_2511_07035_b200 as G
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device"
    return G


def guard_failures(traj, lo=0, hi=None):
    """Element updates of the trajectory (restricted to [lo, hi)) whose m' or v' leaves the guard."""
    bad = 0
    for (_, m, v) in traj[1:]:
        m, v = np.abs(m[lo:hi].astype(np.float64)), np.abs(v[lo:hi].astype(np.float64))
        bad += int(np.count_nonzero(~((m >= M_LO) & (m <= M_HI) & (v >= V_LO) & (v <= V_HI))))
    return bad


def replay_guard_failures(traj, parts, K):
    """Guard failures among the replay's element updates: part j (1-based) gets t0+j .. t0+K-1."""
    bad = 0
    for j in range(1, K):
        lo, hi = parts[j - 1]
        bad += guard_failures([None] + traj[j:K], lo, hi)
    return bad


def run_session(G, state, grads, recs, sargs, t0, K, A=1024):
    """One K-step session through the library; every output vs the oracle, bitwise."""
    n = state[0].size
    p, m, v = (up_f32(x) for x in state)
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    ctx = G.GoCkpt(p, m, v, out, **HP, k_min=1, k_max=max(K, 8), part_align=A, eager_replay=False)
    parts = oracle.make_parts(n, K, A)
    g_dev = [up_u16(g) for g in grads]
    ctx.begin_checkpoint(t0, K)
    for i in range(1, K + 1):
        a = sargs[i - 1]
        ctx.submit(i, a["step"], a["adam_t"], a["lr"], g_dev[i - 1], a["grad_scale"], a["skip"])
    torch.cuda.synchronize()
    traj = oracle.trajectory(*state, grads, recs)
    assert_state_equal((down_f32(p), down_f32(m), down_f32(v)), traj[K], "live S(t0+K)")
    assert np.array_equal(out.cpu().numpy().view(np.uint16), oracle.rne_bf16(traj[K][0])), "bf16 working copy"
    ctx.wait_drained()
    st = ctx.staged()
    cap, glog, _ = oracle.capture_session(*state, grads, recs, parts)
    assert_state_equal((st["master"], st["exp_avg"], st["exp_avg_sq"]), oracle.assemble(cap), "staged")
    for i in range(K - 1):
        assert np.array_equal(st["glog"][i], glog[i]), f"glog {i + 1}"
    want = oracle.replay(cap, glog, recs, parts)
    assert_state_equal(want, traj[K - 1], "oracle O2 vs O1")
    # replay_kernel (groups of 8) on the staged bytes
    dP, dM, dV = (torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3))
    dG = torch.empty(max(1, n * (K - 1) + 128 * K), dtype=torch.int16, device="cuda")
    ctx.replay_gpu(dP, dM, dV, dG)
    assert_state_equal((down_f32(dP), down_f32(dM), down_f32(dV)), want, "gpu replay")
    ck = ctx.finalize()
    assert_state_equal((ck.master, ck.exp_avg, ck.exp_avg_sq), want, "host replay")
    ctx.release()
    ctx.close()
    return traj, parts


def _steps(t0, K, count0, lr=1e-3, gs=lambda s: 1.0):
    recs, sargs = [], []
    for i in range(1, K + 1):
        s, t = t0 + i, count0 + i
        recs.append(oracle.make_step_record(t=t, lr=lr, grad_scale=gs(s), **HP))
        sargs.append(dict(step=s, adam_t=t, lr=lr, grad_scale=gs(s), skip=False))
    return recs, sargs


@pytest.mark.parametrize("n", [(1 << 18) + 4101, (1 << 20) + 2048 * 3 + 17])
def test_cold_start_session(G, n):
    """t0 = 0 from S(0) (m = v = 0): update 1 makes m' = v' = 0 wherever g = 0 (~1.6% of elements)."""
    K, t0, seed = 4, 0, 5
    state = gi.cold_state(seed, n)
    grads = [gi.grad_bits(seed, t0 + i, n, mode=gi.GRAD_LLM, zero_per_256=4) for i in range(1, K + 1)]
    recs, sargs = _steps(t0, K, 0)
    traj, parts = run_session(G, state, grads, recs, sargs, t0, K)
    # the fused kernel's updates (all K) and the replay's (parts 1..K-1) both left the guard
    assert guard_failures(traj) > 1000
    assert replay_guard_failures(traj, parts, K) > 1000


def _planted(seed, n, K, t0):
    """Warm state with planted out-of-range lanes (one lane per group) at tiles, part boundaries and
    the ragged tail; the planted lanes get g = 0 at every step (so tiny moments stay tiny)."""
    p, m, v = gi.warm_state(seed, n)
    grads = [gi.grad_bits(seed, t0 + i, n) for i in range(1, K + 1)]
    rng = np.random.default_rng(seed)
    pos = np.unique(np.concatenate([rng.integers(0, n, 4000), np.arange(n - 64, n),
                                    np.arange(0, n, 2048 * 7 + 3), [n // 4, n // 4 + 1, n // 2 - 1, n // 2]]))
    pos = pos[np.diff(np.concatenate([[-8], pos])) >= 8]  # at most one planted lane per 8-group
    kinds = [("m", 0.0), ("m", np.float32(2.0 ** -140)), ("m", 2.0 ** -45), ("m", -2.0 ** -45), ("m", 2.0 ** 25),
             ("m", -2.0 ** 25), ("v", 0.0), ("v", np.float32(3.0 * 2.0 ** -140)), ("mv", 0.0), ("g", 64.0)]
    for k, e in enumerate(pos):
        what, val = kinds[k % len(kinds)]
        if "m" in what:
            m[e] = val
        if "v" in what:
            v[e] = val
        if what == "g":  # g = 64 at session step 2: |m'| > 2^20 when that step's grad_scale is 2^20
            grads[1][e] = 0x4280
        elif not (what == "m" and abs(val) > 1):
            for g in grads:
                g[e] = 0
    return (p, m, v), grads


@pytest.mark.parametrize("gs_big", [False, True])
def test_planted_out_of_range_lanes(G, gs_big):
    n, K, t0, seed = (1 << 19) + 1000, 4, 40, 9
    state, grads = _planted(seed, n, K, t0)
    # grad_scale 2^20 at session step 2 (a loss-scale unscaling factor applied in the update)
    recs, sargs = _steps(t0, K, t0, gs=(lambda s: 2.0 ** 20 if s == t0 + 2 else 1.0) if gs_big else (lambda s: 1.0))
    traj, parts = run_session(G, state, grads, recs, sargs, t0, K)
    assert guard_failures(traj) > 100
    assert replay_guard_failures(traj, parts, K) > 100


@pytest.mark.parametrize("K,skips", [(4, (3,)), (8, (7,)), (8, (5, 6, 7)), (8, (1, 2)), (6, (1, 3, 5)),
                                     (8, (2, 3, 4, 5, 6, 7))])
def test_replay_kernel_compaction_with_skipped_updates(G, K, skips):
    """The replay kernel keeps only the non-skipped StepRecords (compacted on the host; part j needs the
    compacted records from first[j] on). Skipped updates at the end of the session leave whole stale
    parts with nothing pending (the kernel must not load or store them), skips at the start shift every
    part's first record. The GPU replay (and the host replay) == the synchronous snapshot == oracle O1.
    skips are session steps i (training step t0 + i); the bias-correction count does not advance."""
    n, t0, seed = (1 << 18) + 2048 * 5 + 64, 30, 13
    state = gi.warm_state(seed, n)
    grads = [gi.grad_bits(seed, t0 + i, n) for i in range(1, K + 1)]
    recs, sargs, t = [], [], t0
    for i in range(1, K + 1):
        sk = i in skips
        if not sk:
            t += 1
        gs = 0.5 if i % 3 == 0 else 1.0
        recs.append(oracle.make_step_record(t=t, lr=1e-3, grad_scale=gs, skip=sk, **HP))
        sargs.append(dict(step=t0 + i, adam_t=max(t, 1), lr=1e-3, grad_scale=gs, skip=sk))
    traj, parts = run_session(G, state, grads, recs, sargs, t0, K, A=64)
    assert len(parts) == K
