"""Full-size parity (-m gpu): BASELINE.json's configs at their real shard sizes, in the launch
configuration bench.py times (TMA fused kernel, R=2 ring, copy-engine drain, eager host replay).

The whole checkpoint is compared bitwise with the GPU's own synchronous snapshot S(T); the
oracle (which cannot run 124M-element sessions in seconds) checks sampled windows that cover
every part boundary, the ragged tail and random offsets — exact because the update is
elementwise and the only cross-element inputs are the per-step scalars.
"""

import numpy as np
import pytest
import torch

import gockpt_inputs as gi
import oracle
from gpu_helpers import HP, down_f32, assert_state_equal

pytestmark = pytest.mark.gpu

LR = 3e-4


@pytest.fixture(scope="module")
def G():
    from paper_2511_07035_b200 import build as gbuild
    gbuild.build()
    import paper_2511_07035_b200 as G
    assert torch.cuda.is_available()
    return G


def windows(n, parts, seed, width=2048, extra=6):
    rng = np.random.default_rng(seed)
    starts = {0, max(0, n - width)}
    for lo, hi in parts:
        starts.add(max(0, lo - width // 2))
    for _ in range(extra):
        starts.add(int(rng.integers(0, n - width)))
    idx = np.unique(np.concatenate([np.arange(s, min(n, s + width)) for s in sorted(starts)]))
    return idx.astype(np.uint64)


def run_fullsize(G, n, K, t0, seed, copy_mode="ce", check_staged=False):
    dev = torch.device("cuda", 0)
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m, v = torch.empty_like(p), torch.empty_like(p)
    out = torch.empty(n, dtype=torch.int16, device=dev)
    G.h_generate(G.GEN_MASTER, p, seed, 0, 0, gi.MASTER_FLAT)
    G.h_generate(G.GEN_EXP_AVG, m, seed)
    G.h_generate(G.GEN_EXP_AVG_SQ, v, seed)
    g = torch.empty(n, dtype=torch.int16, device=dev)
    ctx = G.GoCkpt(p, m, v, out, **HP, k_min=K, k_max=K, part_align=1024, copy_mode=copy_mode,
                   eager_replay=not check_staged)
    parts = G.plan_parts(n, K, 1024)
    ctx.begin_checkpoint(t0, K)
    snap = None
    for i in range(1, K + 1):
        s = t0 + i
        G.h_generate(G.GEN_GRAD, g, seed, s, 0, gi.GRAD_LLM, 4)
        if i == K:
            snap = ctx.sync_snapshot()
        ctx.submit(i, s, s, LR, g)
    torch.cuda.synchronize()
    live = (down_f32(p), down_f32(m), down_f32(v))
    staged = None
    if check_staged:
        ctx.wait_drained()
        st = ctx.staged()
        staged = {k: (np.array(v_, copy=True) if isinstance(v_, np.ndarray) else v_) for k, v_ in st.items()
                  if k in ("master", "exp_avg", "exp_avg_sq")}
        staged["glog"] = [x.copy() for x in st["glog"]]
    ck = ctx.finalize()
    ckpt = (ck.master.copy(), ck.exp_avg.copy(), ck.exp_avg_sq.copy())
    assert ck.step == t0 + K - 1
    stats = ctx.stats()
    ctx.release()
    ctx.close()
    return parts, snap, live, ckpt, staged, stats


def oracle_windows(idx, t0, K, seed):
    p0, m0, v0 = gi.warm_state(seed, idx)
    grads = [gi.grad_bits(seed, t0 + i, idx) for i in range(1, K + 1)]
    recs = [oracle.make_step_record(t=t0 + i, lr=LR, **HP) for i in range(1, K + 1)]
    traj = oracle.trajectory(p0, m0, v0, grads, recs)
    return traj, grads


@pytest.mark.parametrize("copy_mode", ["ce", "zerocopy"])
def test_gpt2_small_k8_fullsize(G, copy_mode):
    n, K, t0, seed = 124_439_808, 8, 100, 42
    parts, snap, live, ckpt, staged, stats = run_fullsize(G, n, K, t0, seed, copy_mode, check_staged=True)
    assert_state_equal(ckpt, snap, "checkpoint vs sync snapshot (all elements)")
    idx = windows(n, parts, seed)
    traj, grads = oracle_windows(idx, t0, K, seed)
    ii = idx.astype(np.int64)
    assert_state_equal(tuple(x[ii] for x in ckpt), traj[K - 1], "checkpoint vs oracle S(T) (windows)")
    assert_state_equal(tuple(x[ii] for x in live), traj[K], "live vs oracle S(t0+K) (windows)")
    # staged (pre-replay) bytes vs the oracle's capture on the windows
    for i, (lo, hi) in enumerate(parts):
        sel = (ii >= lo) & (ii < hi)
        want = tuple(x[sel] for x in traj[i])
        got = tuple(staged[k][ii[sel]] for k in ("master", "exp_avg", "exp_avg_sq"))
        assert_state_equal(got, want, f"staged part {i + 1}")
        if i < K - 1:
            selg = ii < hi
            assert np.array_equal(staged["glog"][i][ii[selg]], grads[i][selg])
    assert stats["d2h_bytes"] == oracle.session_bytes(parts)


def test_llama2_7b_zero1_rank_shard_fullsize(G):
    # configs[2]: Llama-2 7B ZeRO-1 over 8 ranks -> one rank's shard, n_r = 842,301,952
    n, K, t0, seed = 842_301_952, 8, 200, 7
    parts, snap, live, ckpt, _, stats = run_fullsize(G, n, K, t0, seed)
    assert_state_equal(ckpt, snap, "7B shard: checkpoint vs sync snapshot (all elements)")
    idx = windows(n, parts, seed, width=1024, extra=4)
    traj, _ = oracle_windows(idx, t0, K, seed)
    assert_state_equal(tuple(x[idx.astype(np.int64)] for x in ckpt), traj[K - 1], "7B shard vs oracle (windows)")
    assert stats["d2h_bytes"] == oracle.session_bytes(parts)


@pytest.mark.parametrize("impl,cfg", [("auto", "default"), ("t", "default"), ("t", "6,1,8"), ("t", "3,2,16"),
                                      ("x", "4,2,16"), ("x", "3,4,16")])
def test_tma_kernel_stress_vs_simple_kernel(G, impl, cfg, monkeypatch):
    """Differential stress at the bench size: the TMA-pipelined fused kernels (the bulk-store default and
    the STG-store variant, several stage configurations) against
    the plain grid-stride kernel (itself bit-exact against the oracle in test_gpu_parity), 24 steps
    plain + session, every element compared bitwise after every step. Catches shared-memory ring
    races (a stage refilled before every lane has read it) that window sampling can miss."""
    import subprocess
    import sys
    import os
    env = dict(os.environ)
    if cfg != "default":
        env["GCK_TMAST_CFG" if impl == "x" else "GCK_TMA_CFG"] = cfg
    env["GCK_TEST_IMPL"] = impl      # auto = the default (bulk stores), t = STG stores, x = bulk stores
    code = r'''
import os, sys, torch
sys.path.insert(0, ".")
import paper_2511_07035_b200 as G
n = 124_439_808
def mk():
    p = torch.empty(n, dtype=torch.float32, device="cuda"); m = torch.empty_like(p); v = torch.empty_like(p)
    G.h_generate(1, p, 5, 0, 0, 0); G.h_generate(2, m, 5); G.h_generate(3, v, 5)
    return p, m, v, torch.empty(n, dtype=torch.int16, device="cuda")
a, b = mk(), mk()
g = torch.empty(n, dtype=torch.int16, device="cuda")
for s in range(1, 25):
    G.h_generate(4, g, 5, s, 0, 1, 4)
    r = G.make_step_record(0.9, 0.999, 1e-8, 0.01, 100 + s, 3e-4)
    if os.environ["GCK_TEST_IMPL"] != "auto":
        os.environ["GCK_FUSED_IMPL"] = os.environ["GCK_TEST_IMPL"]
    else:
        os.environ.pop("GCK_FUSED_IMPL", None)
    G.adamw_step(r, *a[:3], g, a[3])                       # default launcher (TMA at this size) or x
    os.environ["GCK_FUSED_IMPL"] = "simple"
    G.adamw_step(r, *b[:3], g, b[3])                       # reference: the plain grid-stride kernel
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x.view(torch.int32) if x.dtype == torch.float32 else x,
                           y.view(torch.int32) if y.dtype == torch.float32 else y), ("step", s)
print("ok")
'''
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
