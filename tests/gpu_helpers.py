"""Shared helpers of the -m gpu tests (test plumbing only: uploads, comparisons)."""

import numpy as np
import torch

import gockpt_inputs as gi
import oracle

HP = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


def up_f32(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def up_u16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).view(np.int16)).cuda()


def down_f32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.float32, copy=False)


def down_u16(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def max_rel(a: np.ndarray, b: np.ndarray) -> float:
    """Reading R14: |a-b| / max(|a|,|b|), 0 where a == b (incl. +-0)."""
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    den = np.maximum(np.abs(a64), np.abs(b64))
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.where(a64 == b64, 0.0, np.abs(a64 - b64) / den)
    return float(r.max()) if r.size else 0.0


def assert_state_equal(got, want, what=""):
    """Bitwise equality of (master, m, v); on failure report the max relative error (bar: 1e-6)."""
    for name, g, w in zip(("master", "exp_avg", "exp_avg_sq"), got, want):
        g = np.asarray(g, np.float32)
        w = np.asarray(w, np.float32)
        assert g.shape == w.shape, (what, name)
        if not np.array_equal(g.view(np.uint32), w.view(np.uint32)):
            bad = np.flatnonzero(g.view(np.uint32) != w.view(np.uint32))
            raise AssertionError(f"{what} {name}: {bad.size} elements differ (first {bad[:5]}), "
                                 f"max rel {max_rel(g, w):.3e}")
        assert max_rel(g, w) <= 1e-6


def session_inputs(seed, n, K, t0, mode=gi.GRAD_LLM, skips=(), lr0=1e-3):
    """S(t0) (a warm synthetic state), the K session gradients and the oracle StepRecords."""
    p0, m0, v0 = gi.warm_state(seed, n)
    recs, steps = [], []
    t = t0
    for i in range(1, K + 1):
        s = t0 + i
        sk = s in skips
        if not sk:
            t += 1
        lr = lr0 * (1 + 0.01 * s)
        gs = 0.5 if s % 3 == 0 else 1.0
        recs.append(oracle.make_step_record(t=t, lr=lr, grad_scale=gs, skip=sk, **HP))
        steps.append(dict(step=s, adam_t=max(t, 1), lr=lr, grad_scale=gs, skip=sk))
    grads = [gi.grad_bits(seed, t0 + i, n, mode=mode) for i in range(1, K + 1)]
    return (p0, m0, v0), grads, recs, steps
