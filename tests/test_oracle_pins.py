"""Pins of the oracle's update formula against things other than itself (-m "not gpu").

Each test names what fixes the expected value: SPEC's worked scalars,
the hand-worked K=2 fixture (tests/golden/k2_example.txt), a float64 closed
form, torch.optim.AdamW in float64 (library routine), torch's bf16 casts.
"""

import dataclasses
import os

import numpy as np
import pytest
import torch

from oracle import adamw_update, make_step_record, rne_bf16, bf16_to_f32, trajectory, oracle_session
import gockpt_inputs as gi

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "k2_example.txt")


def f32(*xs):
    return np.array(xs, dtype=np.float32)


def bf(*xs):
    return rne_bf16(f32(*xs))


def load_golden(path):
    out = {}
    with open(path) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, *vals = line.split()
            out[k] = [float(x) for x in vals]
    return out


# ---------------------------------------------------------------- SPEC S:73-75
def test_spec_zero_gradient_is_identity():
    # g=0, m=v=0, weight_decay=0 -> master unchanged, m=v remain 0
    rec = make_step_record(0.9, 0.999, 1e-8, 0.0, t=1, lr=1e-3)
    p, m, v, w = adamw_update(f32(1.0, -2.5, 3e-3), f32(0, 0, 0), f32(0, 0, 0), bf(0, 0, 0), rec)
    assert np.array_equal(p, f32(1.0, -2.5, 3e-3))
    assert np.array_equal(m, f32(0, 0, 0)) and np.array_equal(v, f32(0, 0, 0))
    assert np.array_equal(w, rne_bf16(f32(1.0, -2.5, 3e-3)))


def test_spec_pure_decay():
    # g=0, m=v=0, wd=0.01, lr=0.001, w=1.0 -> w' = 1 - 1e-5 = 0.99999
    rec = make_step_record(0.9, 0.999, 1e-8, 0.01, t=1, lr=1e-3)
    p, m, v, _ = adamw_update(f32(1.0), f32(0), f32(0), bf(0), rec)
    assert abs(float(p[0]) - 0.99999) <= 1e-7          # binary32 of 0.99999 +- 1 ulp
    assert float(p[0]) == float(np.float32(1.0) - np.float32(1e-3) * np.float32(0.01))


def test_spec_first_step_unit_gradient():
    # g=1, m=v=0, t=1, b1=.9, b2=.999, eps=1e-8, wd=0, lr=1e-3, w=1 -> m=0.1, v=0.001, w'~0.999
    rec = make_step_record(0.9, 0.999, 1e-8, 0.0, t=1, lr=1e-3)
    p, m, v, _ = adamw_update(f32(1.0), f32(0), f32(0), bf(1.0), rec)
    assert m[0] == np.float32(0.1) and v[0] == np.float32(0.001)
    assert abs(float(p[0]) - 0.999) <= 1e-6            # S:75 "checked within 1e-6"
    # the bias-corrected moments are exactly 1 (m/bc1 = 0.1f/0.1f, v/bc2 = 0.001f/0.001f)
    assert rec.c1 == rec.bc1 and rec.c2 == rec.bc2


def test_scalars_rounded_once_from_binary64():
    # Reading R7: c1 = f32(1 - 0.9) = 0.1f, not f32(1) - f32(0.9) = 0.100000024f
    rec = make_step_record(0.9, 0.999, 1e-8, 0.01, t=3, lr=1e-3)
    assert rec.c1 == np.float32(0.1)
    assert rec.c1 != np.float32(1.0) - np.float32(0.9)
    assert rec.bc1 == np.float32(1 - 0.9 * 0.9 * 0.9)
    assert rec.bc2 == np.float32(1 - 0.999 * 0.999 * 0.999)


# ---------------------------------------------------------------- golden K=2
def test_hand_worked_k2():
    g = load_golden(GOLDEN)
    hp = dict(beta1=g["beta1"][0], beta2=g["beta2"][0], eps=g["eps"][0], weight_decay=g["wd"][0])
    recs = [make_step_record(t=t, lr=g["lr"][0], **hp) for t in (1, 2)]
    # the scalars of the fixture's header are exact
    assert (recs[0].c1, recs[0].c2, recs[0].bc1, recs[0].bc2) == (0.5, 0.25, 0.5, 0.25)
    assert (recs[1].bc1, recs[1].bc2) == (0.75, 0.4375)
    G1, G2 = rne_bf16(f32(*g["G1"])), rne_bf16(f32(*g["G2"]))
    states = trajectory(f32(*g["S0_master"]), f32(*g["S0_m"]), f32(*g["S0_v"]), [G1, G2], recs)
    for k in (1, 2):
        for j, name in enumerate(("master", "m", "v")):
            assert np.array_equal(states[k][j], f32(*g[f"S{k}_{name}"])), (k, name)
    # the session: t0 = 1, K = 2; session steps drive updates 2 and 3 (G(3) never recorded)
    G3 = rne_bf16(f32(7.0, -3.0))
    rec3 = make_step_record(t=3, lr=g["lr"][0], **hp)
    (ck_p, ck_m, ck_v), cap, glog, parts, _ = oracle_session(
        states[1][0], states[1][1], states[1][2], [G2, G3], [recs[1], rec3], K=2)
    assert parts == [(0, 1), (1, 2)]
    assert np.array_equal(np.concatenate(cap[0]), f32(*g["cap1"]))
    assert np.array_equal(bf16_to_f32(glog[0]), f32(*g["glog1"]))
    assert np.array_equal(np.concatenate(cap[1]), f32(*g["cap2"]))
    assert len(glog) == 1
    assert np.array_equal(ck_p, f32(*g["ckpt_master"]))
    assert np.array_equal(ck_m, f32(*g["ckpt_m"]))
    assert np.array_equal(ck_v, f32(*g["ckpt_v"]))
    # negative control: without the replay, elem0 keeps its captured S(1) values
    assert np.array_equal(np.concatenate(cap[0]), f32(*g["noreplay_elem0"]))
    assert not np.array_equal(f32(*g["noreplay_elem0"]), f32(ck_p[0], ck_m[0], ck_v[0]))


# ---------------------------------------------------------------- float64 closed form
@pytest.mark.parametrize("gval", [0.5, -0.03125, 1.5e-4])
def test_constant_gradient_closed_form(gval):
    # m0=v0=0, constant g:  mh_t = g and vh_t = g^2 exactly (bias correction), so
    # p_t = a^t p0 - lr*u*(1-a^t)/(1-a), a = 1 - lr*wd, u = g/(|g|+eps).
    lr, wd, eps, T = 1e-3, 0.01, 1e-8, 60
    gb = rne_bf16(f32(gval))
    gexact = float(bf16_to_f32(gb)[0])
    p = f32(0.75, -1.25)
    m = v = f32(0, 0)
    for t in range(1, T + 1):
        p, m, v, _ = adamw_update(p, m, v, np.repeat(gb, 2), make_step_record(0.9, 0.999, eps, wd, t=t, lr=lr))
    a = 1.0 - lr * wd
    u = gexact / (abs(gexact) + eps)
    for p0, pt in zip((0.75, -1.25), p):
        expect = a ** T * p0 - lr * u * (1 - a ** T) / (1 - a)
        assert abs(float(pt) - expect) <= 2e-6 * max(1.0, abs(expect)), (float(pt), expect)
    # the moments follow their own closed forms: m_T = (1-b1^T) g, v_T = (1-b2^T) g^2
    assert np.allclose(m, (1 - 0.9 ** T) * gexact, rtol=1e-5)
    assert np.allclose(v, (1 - 0.999 ** T) * gexact ** 2, rtol=1e-5)


# ---------------------------------------------------------------- torch.optim.AdamW, float64
@pytest.mark.parametrize("seed,gs", [(42, 1.0), (7, 0.5)])
def test_matches_torch_adamw_float64(seed, gs):
    n, T = 4096, 25
    lr, b1, b2, eps, wd = 1e-3, 0.9, 0.999, 1e-8, 0.01
    p32 = gi.master(seed, n)
    m32 = np.zeros(n, np.float32)
    v32 = np.zeros(n, np.float32)
    w = torch.tensor(p32.astype(np.float64), requires_grad=True)
    opt = torch.optim.AdamW([w], lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd, foreach=False, fused=False)
    for t in range(1, T + 1):
        g = gi.grad_bits(seed, t, n, mode=gi.GRAD_UNIFORM if t % 2 else gi.GRAD_LLM)
        p32, m32, v32, _ = adamw_update(p32, m32, v32, g, make_step_record(b1, b2, eps, wd, t=t, lr=lr, grad_scale=gs))
        w.grad = torch.tensor(bf16_to_f32(g).astype(np.float64) * np.float64(np.float32(gs)))
        opt.step()
    st = opt.state[w]
    ref_p, ref_m, ref_v = w.detach().numpy(), st["exp_avg"].numpy(), st["exp_avg_sq"].numpy()
    # binary32 vs binary64 of the same algebra: a few ulp per step, well inside 1e-5 relative
    assert np.max(np.abs(p32 - ref_p) / np.maximum(np.abs(ref_p), 1e-3)) < 1e-5
    assert np.max(np.abs(m32 - ref_m)) < 1e-5 * np.max(np.abs(ref_m))
    assert np.max(np.abs(v32 - ref_v) / ref_v) < 1e-5
    # the bound discriminates: a plausible slip (bias correction dropped) lands far outside it
    pb, mb, vb = gi.master(seed, n), np.zeros(n, np.float32), np.zeros(n, np.float32)
    for t in range(1, T + 1):
        g = gi.grad_bits(seed, t, n, mode=gi.GRAD_UNIFORM if t % 2 else gi.GRAD_LLM)
        rec = dataclasses.replace(make_step_record(b1, b2, eps, wd, t=t, lr=lr, grad_scale=gs),
                                  bc1=np.float32(1), bc2=np.float32(1))
        pb, mb, vb, _ = adamw_update(pb, mb, vb, g, rec)
    assert np.max(np.abs(pb - ref_p) / np.maximum(np.abs(ref_p), 1e-3)) > 1e-4


# ---------------------------------------------------------------- bf16 conversions
def test_rne_bf16_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(100000).astype(np.float32) * np.float32(3.0),
        (rng.integers(0, 1 << 32, 100000, dtype=np.uint64).astype(np.uint32)).view(np.float32),
        # exact ties: low 16 bits 0x8000, both parities of bit 16
        (np.arange(0x3F800000, 0x3F800000 + (1 << 20), 1 << 15, dtype=np.uint32) | np.uint32(0x8000)).view(np.float32),
        f32(0.0, -0.0, np.inf, -np.inf, 1e-40, -1e-40, 3.4e38),
    ])
    x = x[np.isfinite(x) | np.isinf(x)]
    ref = torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(rne_bf16(x), ref)
    assert rne_bf16(f32(np.nan))[0] == 0x7FC0


def test_bf16_widening_matches_torch():
    bits = np.arange(0, 1 << 16, dtype=np.uint32).astype(np.uint16)
    ref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    got = bf16_to_f32(bits)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
