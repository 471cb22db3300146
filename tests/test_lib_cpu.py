"""libgockpt.so on the CPU host (-m "not gpu"): it loads, exports every symbol the
header declares with the struct layouts the binding assumes, and its host-only
building blocks (a0 StepRecord, a1 plan, a5 host replay) agree with the oracle
bit for bit. No GPU compute is called here."""

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import gockpt_inputs as gi
import oracle
from paper_2511_07035_b200 import build as gbuild

HP = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


@pytest.fixture(scope="module")
def G(repo_root):
    gbuild.build()
    import paper_2511_07035_b200 as G
    return G


def header_functions(root):
    text = open(os.path.join(root, "include", "gockpt.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gck_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(G, repo_root):
    from paper_2511_07035_b200._lib import SIGNATURES
    names = header_functions(repo_root)
    assert len(names) >= 20
    L = G.lib()
    for name in names:
        assert hasattr(L, name), name
        assert name in SIGNATURES, name
    assert set(SIGNATURES) == set(names)
    out = subprocess.run(["nm", "-D", "--defined-only", G.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gck_\w+)", out))
    assert set(names) <= exported


def test_struct_layouts_match_c(G, repo_root, tmp_path):
    from paper_2511_07035_b200 import _lib as L
    structs = {"gck_hparams": L.Hparams, "gck_config": L.Config, "gck_tensors": L.Tensors,
               "gck_step_args": L.StepArgs, "gck_step_record": L.StepRecord, "gck_checkpoint": L.Checkpoint,
               "gck_staged": L.Staged, "gck_stats": L.Stats, "gck_file_header": L.FileHeader,
               "gck_persist_stats": L.PersistStats, "gck_log_header": L.LogHeader,
               "gck_session_step": L.SessionStep}
    src = tmp_path / "sz.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gockpt.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(repo_root, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)


def test_no_device_here_and_create_fails_loudly(G):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    assert G.device_count() == 0
    from paper_2511_07035_b200 import _lib as L
    cfg = L.Config(L.ABI_VERSION, 0, 1024, 1, 4, 8, 2, 0, 0, 0, 0, 0, 1, 1)
    hp = L.Hparams(0.9, 0.999, 1e-8, 0.01)
    t = L.Tensors(4096, 8192, 12288, None)     # fake, aligned, never dereferenced
    ctx = C.c_void_p()
    st = G.lib().gck_create(C.byref(cfg), C.byref(hp), C.byref(t), C.byref(ctx))
    assert st == L.E_NODEVICE and not ctx.value


def test_create_validation_errors(G):
    from paper_2511_07035_b200 import _lib as L
    hp = L.Hparams(0.9, 0.999, 1e-8, 0.01)
    t = L.Tensors(4096, 8192, 12288, None)
    ctx = C.c_void_p()
    bad = [
        L.Config(L.ABI_VERSION + 7, 0, 1024, 1, 4, 8, 2, 0, 0, 0, 0, 0, 1, 1),   # ABI
        L.Config(L.ABI_VERSION, 0, 0, 1, 4, 8, 2, 0, 0, 0, 0, 0, 1, 1),          # n = 0
        L.Config(L.ABI_VERSION, 0, 1024, 1, 4, 12, 2, 0, 0, 0, 0, 0, 1, 1),      # A % 8 != 0
        L.Config(L.ABI_VERSION, 0, 1024, 5, 4, 8, 2, 0, 0, 0, 0, 0, 1, 1),       # k_min > k_max
        L.Config(L.ABI_VERSION, 0, 1024, 1, 65, 8, 2, 0, 0, 0, 0, 0, 1, 1),      # k_max > 64
        L.Config(L.ABI_VERSION, 0, 1024, 1, 4, 8, 3, 0, 0, 0, 0, 0, 1, 1),       # R = 3
        L.Config(L.ABI_VERSION, 0, 64, 9, 9, 8, 2, 0, 0, 0, 0, 0, 1, 1),         # k_min > ceil(n/A)
        L.Config(L.ABI_VERSION, 0, 1024, 1, 4, 8, 2, 0, 0, 0, 0, 0, 1, 1, plan=2),  # bad plan
    ]
    for cfg in bad:
        assert G.lib().gck_create(C.byref(cfg), C.byref(hp), C.byref(t), C.byref(ctx)) == L.E_INVALID
    cfg = L.Config(L.ABI_VERSION, 0, 1024, 1, 4, 8, 2, 0, 0, 0, 0, 0, 1, 1)
    t_mis = L.Tensors(4100, 8192, 12288, None)                                     # misaligned master
    assert G.lib().gck_create(C.byref(cfg), C.byref(hp), C.byref(t_mis), C.byref(ctx)) == L.E_INVALID
    assert b"aligned" in G.lib().gck_last_error(None)


# ---------------------------------------------------------------- a0
@pytest.mark.parametrize("t", [1, 2, 3, 10, 100, 1000, 12345])
@pytest.mark.parametrize("lr,gs", [(1e-3, 1.0), (3e-4, 0.5), (0.25, 1 / 3)])
def test_step_record_matches_oracle(G, t, lr, gs):
    r = G.make_step_record(0.9, 0.999, 1e-8, 0.01, t, lr, gs)
    o = oracle.make_step_record(0.9, 0.999, 1e-8, 0.01, t=t, lr=lr, grad_scale=gs)
    for f in ("b1", "c1", "b2", "c2", "bc1", "bc2", "lr", "eps", "wd", "gs"):
        assert np.float32(getattr(r, f)) == getattr(o, f), f
    assert r.t == t and r.skip == 0


def test_step_record_errors(G):
    from paper_2511_07035_b200 import _lib as L
    rec = L.StepRecord()
    hp = L.Hparams(0.9, 0.999, 1e-8, 0.01)
    assert G.lib().gck_make_step_record(C.byref(hp), 0, 1e-3, 1.0, 0, C.byref(rec)) == L.E_INVALID
    assert G.lib().gck_make_step_record(C.byref(hp), 0, 1e-3, 1.0, 1, C.byref(rec)) == L.OK


# ---------------------------------------------------------------- a1
@pytest.mark.parametrize("n,K,A", [(10, 3, 1), (10, 1, 1), (7, 7, 1), (2 ** 20, 4, 1024), (1_000_003, 4, 1024),
                                   (124_439_808, 8, 1024), (3 * 1024 + 1, 4, 1024), (999, 64, 8)])
def test_plan_parts_matches_oracle(G, n, K, A):
    assert G.plan_parts(n, K, A) == oracle.make_parts(n, K, A)


@pytest.mark.parametrize("n,K,A", [(10, 3, 1), (10, 1, 1), (7, 7, 1), (2 ** 20, 4, 1024), (1_000_003, 4, 1024),
                                   (124_439_808, 8, 1024), (3 * 1024 + 1, 4, 1024), (999, 64, 8),
                                   (3_253_966_336, 16, 1024), (6_507_932_160, 16, 1024), (842_301_952, 64, 1024),
                                   (4096, 2, 1), (13, 5, 2)])
def test_plan_parts_balanced_matches_oracle(G, n, K, A):
    # DESIGN.md R17: bit-identical plan (same integer rule); never a larger V_max than the equal plan
    got = G.plan_parts(n, K, A, plan="balanced")
    assert got == oracle.make_parts_balanced(n, K, A)
    assert oracle.max_slot_bytes(got) <= oracle.max_slot_bytes(oracle.make_parts(n, K, A))
    assert G.plan_parts(n, K, A, plan="equal") == oracle.make_parts(n, K, A)


def test_plan_parts_balanced_sweep_matches_oracle(G):
    rng = np.random.default_rng(5)
    for _ in range(300):
        A = int(rng.choice([1, 8, 1024]))
        n = int(rng.integers(1, 1 << 24)) if A > 1 else int(rng.integers(1, 5000))
        U = -(-n // A)
        K = int(rng.integers(1, min(U, 64) + 1))
        assert G.plan_parts(n, K, A, plan="balanced") == oracle.make_parts_balanced(n, K, A), (n, K, A)


def test_plan_parts_errors(G):
    from paper_2511_07035_b200 import GckError
    for n, K, A in [(5, 6, 1), (0, 1, 1), (10, 0, 1), (4096, 5, 1024), (10, 65, 1)]:
        with pytest.raises(GckError):
            G.plan_parts(n, K, A)


# ---------------------------------------------------------------- a5 host replay vs oracle (bitwise)
def _session(seed, n, K, t0, A, mode, skips=()):
    p0, m0, v0 = gi.warm_state(seed, n)
    recs, t = [], t0
    for i in range(1, K + 1):
        s = t0 + i
        sk = s in skips
        if not sk:
            t += 1
        recs.append(oracle.make_step_record(t=t, lr=1e-3 * (1 + 0.01 * s), grad_scale=0.5 if s % 3 == 0 else 1.0,
                                            skip=sk, **HP))
    grads = [gi.grad_bits(seed, t0 + i, n, mode=mode) for i in range(1, K + 1)]
    return p0, m0, v0, recs, grads


def _lib_recs(G, orecs):
    out = []
    for r in orecs:
        out.append(G.make_step_record(0.9, 0.999, 1e-8, 0.01, max(r.t, 1), float(r.lr), float(r.gs), r.skip))
    return out


@pytest.mark.parametrize("n,K,A", [(1, 1, 1), (9, 4, 1), (1000, 8, 1), (100_003, 4, 1024), (2 ** 18, 8, 1024),
                                   (65_537, 16, 8)])
@pytest.mark.parametrize("mode", [gi.GRAD_UNIFORM, gi.GRAD_LLM])
@pytest.mark.parametrize("threads", [1, 4])
def test_replay_host_bitwise_vs_oracle(G, n, K, A, mode, threads):
    p0, m0, v0, orecs, grads = _session(42, n, K, 10, A, mode)
    parts = oracle.make_parts(n, K, A)
    cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, orecs, parts)
    want = oracle.replay(cap, glog, orecs, parts)
    p, m, v = (np.ascontiguousarray(x) for x in oracle.assemble(cap))
    lrecs = _lib_recs(G, orecs)
    # the library's records must be the oracle's (lr/gs exact through float32)
    for a, b in zip(lrecs, orecs):
        assert np.float32(a.lr) == b.lr and np.float32(a.bc2) == b.bc2
    G.replay_host(lrecs, parts, p, m, v, [np.ascontiguousarray(g) for g in glog], threads=threads)
    for got, exp in zip((p, m, v), want):
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_replay_host_with_skipped_step(G):
    n, K = 5000, 5
    p0, m0, v0, orecs, grads = _session(7, n, K, 20, 8, gi.GRAD_LLM, skips={23})
    parts = oracle.make_parts(n, K, 8)
    cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, orecs, parts)
    want = oracle.replay(cap, glog, orecs, parts)
    p, m, v = (np.ascontiguousarray(x) for x in oracle.assemble(cap))
    G.replay_host(_lib_recs(G, orecs), parts, p, m, v, glog, threads=3)
    for got, exp in zip((p, m, v), want):
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_replay_host_denormals_kept(G):
    # reading R13: no FTZ/DAZ -- a denormal moment must survive the replay exactly as in the oracle
    import torch
    torch.set_flush_denormal(True)          # the host thread's MXCSR is FTZ/DAZ; workers must clear it
    try:
        n, K = 4096, 3
        p0, m0, v0, orecs, grads = _session(3, n, K, 5, 8, gi.GRAD_LLM)
        m0 = m0.copy()
        m0[: n // 2] = np.float32(1e-39)      # denormal binary32
        v0 = v0.copy()
        v0[:64] = np.float32(2e-40)
        grads = [g.copy() for g in grads]
        for g in grads:
            g[:128] = 0
        parts = oracle.make_parts(n, K, 8)
        cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, orecs, parts)
        want = oracle.replay(cap, glog, orecs, parts)
        p, m, v = (np.ascontiguousarray(x) for x in oracle.assemble(cap))
        for threads in (1, 2):
            pp, mm, vv = p.copy(), m.copy(), v.copy()
            G.replay_host(_lib_recs(G, orecs), parts, pp, mm, vv, glog, threads=threads)
            for got, exp in zip((pp, mm, vv), want):
                assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    finally:
        torch.set_flush_denormal(False)


def test_replay_host_rejects_bad_parts(G):
    from paper_2511_07035_b200 import GckError
    p = np.zeros(10, np.float32)
    recs = [G.make_step_record(0.9, 0.999, 1e-8, 0.01, 1, 1e-3)] * 2
    g = [np.zeros(10, np.uint16)]
    for parts in ([(0, 5), (6, 10)], [(0, 5), (5, 9)], [(1, 5), (5, 10)], [(0, 5), (5, 5)]):
        with pytest.raises(GckError):
            G.replay_host(recs, parts, p, p.copy(), p.copy(), g)


def test_ring_bytes_required(G):
    # R x the largest 256-B-aligned [master_i | m_i | v_i | G[0:hi_i]] slot over K in [k_min, k_max]
    al = lambda x: (x + 255) // 256 * 256
    for n, kmin, kmax, A, R in [(124_439_808, 8, 8, 1024, 2), (1 << 20, 2, 8, 1024, 1), (1000, 1, 4, 8, 2)]:
        best = 0
        for K in range(kmin, kmax + 1):
            parts = oracle.make_parts(n, K, A)
            for i, (lo, hi) in enumerate(parts):
                best = max(best, 3 * al(4 * (hi - lo)) + al(2 * (hi if i < K - 1 else 0)))
        assert G.ring_bytes_required(n, kmin, kmax, A, R) == R * best
    assert G.ring_bytes_required(0, 1, 4) == 0 and G.ring_bytes_required(100, 5, 4) == 0


def test_ring_bytes_required_balanced(G):
    # the same rule over the balanced plans; a smaller ring wherever the plan lowers V_max
    al = lambda x: (x + 255) // 256 * 256
    for n, kmin, kmax, A, R in [(124_439_808, 8, 8, 1024, 2), (3_253_966_336, 2, 16, 1024, 2), (1000, 1, 4, 8, 1)]:
        best = 0
        for K in range(kmin, kmax + 1):
            parts = oracle.make_parts_balanced(n, K, A)
            for i, (lo, hi) in enumerate(parts):
                best = max(best, 3 * al(4 * (hi - lo)) + al(2 * (hi if i < K - 1 else 0)))
        got = G.ring_bytes_required(n, kmin, kmax, A, R, plan="balanced")
        assert got == R * best
        assert got <= G.ring_bytes_required(n, kmin, kmax, A, R)
    assert G.ring_bytes_required(124_439_808, 8, 8, 1024, 2, plan="balanced") < \
        0.8 * G.ring_bytes_required(124_439_808, 8, 8, 1024, 2)


# ---------------------------------------------------------------- a3 drain verification checksum
def _checksum_ref(b: bytes):
    """The definition in include/gockpt.h: little-endian 32-bit words (last one zero-padded),
    A = sum w_i, B = sum (i+1) w_i, mod 2^64 (numpy uint64 arithmetic wraps)."""
    pad = (-len(b)) % 4
    w = np.frombuffer(b + b"\0" * pad, dtype="<u4").astype(np.uint64)
    idx = np.arange(1, w.size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(w.sum(dtype=np.uint64)), int((w * idx).sum(dtype=np.uint64))


@pytest.mark.parametrize("nbytes", [0, 1, 3, 4, 17, 4096, (1 << 26) + 4 * 5 + 2])
def test_checksum_matches_definition(G, nbytes):
    rng = np.random.default_rng(nbytes)
    buf = rng.integers(0, 256, nbytes, dtype=np.uint8)
    assert G.checksum(buf, threads=4) == _checksum_ref(buf.tobytes())
    assert G.checksum(buf, threads=1) == _checksum_ref(buf.tobytes())


def test_checksum_detects_flip_and_swap(G):
    rng = np.random.default_rng(1)
    buf = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    ref = G.checksum(buf)
    for pos in (0, 1, 12345, (1 << 20) - 1):
        for bit in range(8):
            b2 = buf.copy()
            b2[pos] ^= np.uint8(1 << bit)
            assert G.checksum(b2)[0] != ref[0]          # any single corrupted byte changes A
    w = buf.view(np.uint32).copy()
    w[[10, 11]] = w[[11, 10]]                            # transposed words keep A, change B
    if w[10] != w[11]:
        got = G.checksum(w)
        assert got[0] == ref[0] and got[1] != ref[1]
