"""O1 — plain mixed-precision AdamW (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Paper anchors:
  P:130-134 (§2.1)  each step N updates M^N -> M^{N+1}, O^N -> O^{N+1} from G^N;
                    "learning rate scheduling" is part of the update.
  P:147-149 (§2.2)  16-bit params and gradients; an FP32 master copy; FP32
                    AdamW m and v.
  P:345 (§4.3.1)    "we update parameters on the CPU using the AdamW
                    optimization strategy" (no formula given).
  SPEC S:70         the update written out: m <- b1 m + (1-b1) g; v <- b2 v +
                    (1-b2) g^2; mh = m/(1-b1^t); vh = v/(1-b2^t);
                    w <- w - lr (mh/(sqrt(vh)+eps) + wd w), t = global count.
  SPEC S:96         bias correction with t = global update count.

Readings (DESIGN.md §"Readings of the paper"): R6 op order as written below,
R7 scalars rounded once from binary64, R8 per-step grad_scale and skip.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

F32 = np.float32


@dataclass(frozen=True)
class StepRecord:
    """a0 — the binary32 scalars one update consumes."""
    t: int          # bias-correction count (non-skipped updates up to and including this one)
    skip: bool
    b1: np.float32
    c1: np.float32
    b2: np.float32
    c2: np.float32
    bc1: np.float32
    bc2: np.float32
    lr: np.float32
    eps: np.float32
    wd: np.float32
    gs: np.float32


def _pow_running(beta: float, t: int) -> float:
    """beta**t as a left-to-right binary64 running product (reading R7)."""
    acc = 1.0
    for _ in range(t):
        acc = acc * beta
    return acc


def make_step_record(beta1: float, beta2: float, eps: float, weight_decay: float,
                     t: int, lr: float, grad_scale: float = 1.0, skip: bool = False) -> StepRecord:
    """Compute the binary32 scalars of update number t from binary64 hyperparameters.

    Every scalar is formed in binary64 and rounded ONCE to binary32 (reading R7):
    c1 = f32(1 - beta1) (not f32(1) - f32(beta1)), bc1 = f32(1 - beta1**t), ...
    """
    if not skip and t < 1:
        raise ValueError("bias-correction count t must be >= 1 for a non-skipped update")
    tt = max(t, 1)
    return StepRecord(
        t=t, skip=bool(skip),
        b1=F32(beta1), c1=F32(1.0 - beta1),
        b2=F32(beta2), c2=F32(1.0 - beta2),
        bc1=F32(1.0 - _pow_running(beta1, tt)),
        bc2=F32(1.0 - _pow_running(beta2, tt)),
        lr=F32(lr), eps=F32(eps), wd=F32(weight_decay), gs=F32(grad_scale),
    )


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to binary32: bits << 16."""
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def rne_bf16(x: np.ndarray) -> np.ndarray:
    """Round binary32 to bf16 bits, round-to-nearest-even; NaN -> 0x7FC0.

    u = bits(x); (u + 0x7FFF + ((u >> 16) & 1)) >> 16, truncated to 16 bits.
    """
    x = np.asarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) & np.uint64(0xFFFF)
    r = r.astype(np.uint16)
    r[np.isnan(x)] = np.uint16(0x7FC0)
    return r


def adamw_update(p: np.ndarray, m: np.ndarray, v: np.ndarray, g_bits: np.ndarray,
                 rec: StepRecord):
    """One normative mixed-precision AdamW update (returns new arrays).

    Inputs: p, m, v binary32 arrays; g_bits the bf16 gradient (uint16 bits);
    rec the StepRecord. Every line is one correctly-rounded binary32 op:

        g   = f32(g_bits) * gs
        m'  = (b1*m) + (c1*g)
        v'  = (b2*v) + (c2*(g*g))
        mh  = m' / bc1 ;  vh = v' / bc2
        u   = mh / (sqrt(vh) + eps)
        p'  = p - (lr * (u + (wd*p)))
        out = RNE_bf16(p')      (working copy; not part of the checkpoint)

    A skipped step returns the state unchanged (reading R8).
    """
    p = np.asarray(p, dtype=np.float32)
    m = np.asarray(m, dtype=np.float32)
    v = np.asarray(v, dtype=np.float32)
    if rec.skip:
        return p.copy(), m.copy(), v.copy(), rne_bf16(p)
    g = bf16_to_f32(np.asarray(g_bits, dtype=np.uint16))
    g = g * rec.gs
    m_new = (rec.b1 * m) + (rec.c1 * g)
    v_new = (rec.b2 * v) + (rec.c2 * (g * g))
    mh = m_new / rec.bc1
    vh = v_new / rec.bc2
    u = mh / (np.sqrt(vh) + rec.eps)
    p_new = p - (rec.lr * (u + (rec.wd * p)))
    assert p_new.dtype == np.float32 and m_new.dtype == np.float32 and v_new.dtype == np.float32
    return p_new, m_new, v_new, rne_bf16(p_new)


def trajectory(p, m, v, grads, recs):
    """O1: the plain synchronous trajectory. Applies recs[k] with grads[k] in order.

    Returns the list of states [S(start), S(start+1), ...] as (p, m, v) tuples.
    """
    states = [(np.array(p, dtype=np.float32), np.array(m, dtype=np.float32), np.array(v, dtype=np.float32))]
    for g, rec in zip(grads, recs):
        cp, cm, cv = states[-1]
        np_, nm, nv, _ = adamw_update(cp, cm, cv, g, rec)
        states.append((np_, nm, nv))
    return states
