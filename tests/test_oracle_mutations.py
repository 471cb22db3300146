"""The oracle's pins discriminate (-m "not gpu"): each plausible mistake in the oracle's arithmetic
or session logic — applied here as a mutant of the oracle function — fails at least one of the
pins the real oracle passes (SPEC scalars, the hand-worked K=2 golden, the constant-gradient
closed form, torch.optim.AdamW in float64, the K=3 trace, brute force O2 == O1)."""

import dataclasses
import os

import numpy as np
import pytest
import torch

import gockpt_inputs as gi
import oracle
from oracle import adamw as OA

F32 = np.float32
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "k2_example.txt")


def golden():
    out = {}
    for line in open(GOLDEN):
        line = line.split("#", 1)[0].strip()
        if line:
            k, *vals = line.split()
            out[k] = [float(x) for x in vals]
    return out


# ---- mutants of the normative update (same signature as oracle.adamw_update) -------------------
def make_update(kind):
    def upd(p, m, v, g_bits, rec):
        p, m, v = (np.asarray(x, np.float32) for x in (p, m, v))
        if rec.skip:
            return p.copy(), m.copy(), v.copy(), OA.rne_bf16(p)
        g = OA.bf16_to_f32(np.asarray(g_bits, np.uint16)) * rec.gs
        b1, c1, b2, c2 = rec.b1, rec.c1, rec.b2, rec.c2
        if kind == "swap_betas":
            b1, c1, b2, c2 = b2, c2, b1, c1
        m2 = b1 * m + c1 * g
        v2 = b2 * v + c2 * (g * g)
        if kind == "v_uses_abs_g":
            v2 = b2 * v + c2 * np.abs(g)
        mh, vh = m2 / rec.bc1, v2 / rec.bc2
        if kind == "no_bias_correction":
            mh, vh = m2, v2
        d = np.sqrt(vh) + rec.eps
        if kind == "eps_inside_sqrt":
            d = np.sqrt(vh + rec.eps)
        u = mh / d
        p2 = p - rec.lr * (u + rec.wd * p)
        if kind == "decay_sign":
            p2 = p - rec.lr * (u - rec.wd * p)
        if kind == "coupled_l2":             # Adam + L2 (decay folded into g) instead of AdamW
            g2 = g + rec.wd * p
            m2 = b1 * m + c1 * g2
            v2 = b2 * v + c2 * (g2 * g2)
            p2 = p - rec.lr * ((m2 / rec.bc1) / (np.sqrt(v2 / rec.bc2) + rec.eps))
        if kind == "grad_scale_ignored":
            return make_update("none")(p, m, v, g_bits, dataclasses.replace(rec, gs=F32(1)))
        return p2.astype(np.float32), m2.astype(np.float32), v2.astype(np.float32), OA.rne_bf16(p2)
    return upd


def record_mutant(kind):
    def mk(beta1, beta2, eps, weight_decay, t, lr, grad_scale=1.0, skip=False):
        r = OA.make_step_record(beta1, beta2, eps, weight_decay, t=t, lr=lr, grad_scale=grad_scale, skip=skip)
        if kind == "bc_t_minus_1":
            tt = max(t - 1, 1)
            r = dataclasses.replace(r, bc1=F32(1 - beta1 ** tt), bc2=F32(1 - beta2 ** tt))
        if kind == "c_from_f32":
            r = dataclasses.replace(r, c1=F32(1) - F32(beta1), c2=F32(1) - F32(beta2))
        return r
    return mk


# ---- the pins, as predicates over (update, make_record) ---------------------------------------
def pin_spec_scalars(upd, mk):
    rec = mk(0.9, 0.999, 1e-8, 0.0, t=1, lr=1e-3)
    p, m, v, _ = upd(F32([1.0]), F32([0]), F32([0]), OA.rne_bf16(F32([1.0])), rec)
    ok = m[0] == F32(0.1) and v[0] == F32(0.001) and abs(float(p[0]) - 0.999) <= 1e-6
    rec = mk(0.9, 0.999, 1e-8, 0.01, t=1, lr=1e-3)
    p, _, _, _ = upd(F32([1.0]), F32([0]), F32([0]), OA.rne_bf16(F32([0.0])), rec)
    return ok and abs(float(p[0]) - 0.99999) <= 1e-7


def pin_golden_k2(upd, mk):
    g = golden()
    hp = dict(beta1=g["beta1"][0], beta2=g["beta2"][0], eps=g["eps"][0], weight_decay=g["wd"][0])
    recs = [mk(t=t, lr=g["lr"][0], **hp) for t in (1, 2)]
    s = (F32(g["S0_master"]), F32(g["S0_m"]), F32(g["S0_v"]))
    for k, G in ((1, "G1"), (2, "G2")):
        s = upd(*s, OA.rne_bf16(F32(g[G])), recs[k - 1])[:3]
        if not all(np.array_equal(a, F32(g[f"S{k}_{n}"])) for a, n in zip(s, ("master", "m", "v"))):
            return False
    return True


def pin_closed_form(upd, mk):
    lr, wd, eps, T, gval = 1e-3, 0.01, 1e-8, 60, 0.5
    gb = OA.rne_bf16(F32([gval]))
    p, m, v = F32([0.75]), F32([0]), F32([0])
    for t in range(1, T + 1):
        p, m, v, _ = upd(p, m, v, gb, mk(0.9, 0.999, eps, wd, t=t, lr=lr))
    a = 1 - lr * wd
    expect = a ** T * 0.75 - lr * (gval / (gval + eps)) * (1 - a ** T) / (1 - a)
    return abs(float(p[0]) - expect) <= 2e-6


def pin_torch_adamw(upd, mk, gs=0.5):
    n, T = 512, 15
    p32 = gi.master(42, n)
    m32 = np.zeros(n, np.float32)
    v32 = np.zeros(n, np.float32)
    w = torch.tensor(p32.astype(np.float64), requires_grad=True)
    opt = torch.optim.AdamW([w], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, foreach=False)
    for t in range(1, T + 1):
        g = gi.grad_bits(42, t, n, mode=gi.GRAD_UNIFORM)
        p32, m32, v32, _ = upd(p32, m32, v32, g, mk(0.9, 0.999, 1e-8, 0.01, t=t, lr=1e-3, grad_scale=gs))
        w.grad = torch.tensor(OA.bf16_to_f32(g).astype(np.float64) * float(np.float32(gs)))
        opt.step()
    ref = w.detach().numpy()
    st = opt.state[w]
    ref_m, ref_v = st["exp_avg"].numpy(), st["exp_avg_sq"].numpy()
    return (np.max(np.abs(p32 - ref) / np.maximum(np.abs(ref), 1e-3)) < 1e-5
            and np.max(np.abs(m32 - ref_m)) < 1e-5 * np.max(np.abs(ref_m))
            and np.max(np.abs(v32 - ref_v) / ref_v) < 1e-5)


PINS = [pin_spec_scalars, pin_golden_k2, pin_closed_form, pin_torch_adamw]


def test_real_oracle_passes_every_pin():
    for pin in PINS:
        assert pin(oracle.adamw_update, OA.make_step_record), pin.__name__


@pytest.mark.parametrize("kind", ["swap_betas", "v_uses_abs_g", "no_bias_correction", "eps_inside_sqrt",
                                  "decay_sign", "coupled_l2", "grad_scale_ignored"])
def test_update_mutant_is_caught(kind):
    upd = make_update(kind)
    failed = [pin.__name__ for pin in PINS if not pin(upd, OA.make_step_record)]
    assert failed, f"mutant {kind} passes every pin"


@pytest.mark.parametrize("kind", ["bc_t_minus_1", "c_from_f32"])
def test_record_mutant_is_caught(kind):
    failed = [pin.__name__ for pin in PINS if not pin(oracle.adamw_update, record_mutant(kind))]
    assert failed, f"mutant {kind} passes every pin"


# ---- session-logic mutants against the K=3 trace and brute force O2 == O1 ------------------------
def session_mutant(kind):
    def capture(p0, m0, v0, grads, recs, parts):
        K = len(parts)
        p, m, v = (np.array(x, np.float32) for x in (p0, m0, v0))
        cap, glog = [], []
        for i in range(1, K + 1):
            lo, hi = parts[i - 1]
            if kind == "post_update_capture":
                p2, m2, v2, _ = oracle.adamw_update(p, m, v, grads[i - 1], recs[i - 1])
                cap.append((p2[lo:hi].copy(), m2[lo:hi].copy(), v2[lo:hi].copy()))
            else:
                cap.append((p[lo:hi].copy(), m[lo:hi].copy(), v[lo:hi].copy()))
            if i < K:
                ghi = parts[i - 2][1] if (kind == "prefix_off_by_one_part" and i >= 2) else hi
                g = np.array(grads[i - 1][:ghi], np.uint16)
                if kind == "prefix_off_by_one_part" and len(g) < hi:
                    g = np.concatenate([g, np.zeros(hi - len(g), np.uint16)])
                glog.append(g)
            p, m, v, _ = oracle.adamw_update(p, m, v, grads[i - 1], recs[i - 1])
        return cap, glog

    def replay(cap, glog, recs, parts):
        K = len(parts)
        p, m, v = oracle.assemble(cap)
        for j in range(1, K):
            lo, hi = parts[j - 1]
            pj, mj, vj = p[lo:hi], m[lo:hi], v[lo:hi]
            steps = range(j, K)
            if kind == "replay_one_step_short":
                steps = range(j + 1, K)
            if kind == "replay_reversed":
                steps = reversed(list(steps))
            for i in steps:
                pj, mj, vj, _ = oracle.adamw_update(pj, mj, vj, glog[i - 1][lo:hi], recs[i - 1])
            p[lo:hi], m[lo:hi], v[lo:hi] = pj, mj, vj
        return p, m, v
    return capture, replay


@pytest.mark.parametrize("kind", ["post_update_capture", "prefix_off_by_one_part", "replay_one_step_short",
                                  "replay_reversed"])
def test_session_mutant_is_caught(kind):
    capture, replay = session_mutant(kind)
    HP = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    caught = False
    for n, K in [(10, 3), (9, 4), (64, 8)]:
        t0 = 5
        p0, m0, v0 = gi.warm_state(3, n)
        recs = [oracle.make_step_record(t=t0 + i, lr=1e-3, **HP) for i in range(1, K + 1)]
        grads = [gi.grad_bits(3, t0 + i, n) for i in range(1, K + 1)]
        parts = oracle.make_parts(n, K)
        target = oracle.trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]
        cap, glog = capture(p0, m0, v0, grads, recs, parts)
        got = replay(cap, glog, recs, parts)
        if not all(np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(got, target)):
            caught = True
    assert caught, f"session mutant {kind} passes brute force"
