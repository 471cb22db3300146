"""GoCkpt oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the GoCkpt hot path
computes (arXiv 2511.07035, §4.2.1 lines 277-279 and §4.3.1).
It exists so the CUDA path (``paper_2511_07035_b200``) can be checked element
by element. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it. The product path
never imports, links or executes anything in this directory, and this
directory never imports the product path: the two share no code. The one
shared module is ``gockpt_inputs`` (seeded input generators, no method
arithmetic).

Modules
  adamw.py      a0 StepRecord + the normative mixed-precision AdamW update
                (O1: plain synchronous trajectory S(0) -> S(T)).
  partition.py  a1 partition plan (parts, gradient prefixes, byte counts).
  replay.py     O2: the plain K-step partitioned capture + gradient-assisted
                replay, exactly in the paper's order; plus its
                streaming form (updates applied as the slices arrive).

Numerics: every floating-point operation is an IEEE binary32 numpy operation
(round-to-nearest-even, no FMA contraction, denormals kept), in the operation
order written in DESIGN.md "Normative update". Hyperparameter scalars are
computed in binary64 and rounded once to binary32 (reading R7).

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``): SPEC's scalar examples,
the hand-worked K=2 example (tests/golden/k2_example.txt), a float64 closed
form for constant gradients, torch.optim.AdamW in float64, brute force O2==O1
over every contiguous partition of tiny vectors, the paper's K=3 version trace,
SPEC's make_parts examples and closed-form byte counts; the balanced plan against
brute-force minima over every partition and the continuous optimum. No function here is
"parity unpinned".
"""

from .adamw import StepRecord, make_step_record, adamw_update, rne_bf16, bf16_to_f32, trajectory
from .partition import make_parts, make_parts_balanced, max_slot_bytes, grad_prefix, session_bytes, slot_bytes
from .replay import capture_session, replay, replay_streaming, assemble, oracle_session

__all__ = [
    "StepRecord", "make_step_record", "adamw_update", "rne_bf16", "bf16_to_f32", "trajectory",
    "make_parts", "make_parts_balanced", "max_slot_bytes", "grad_prefix", "session_bytes", "slot_bytes",
    "capture_session", "replay", "replay_streaming", "assemble", "oracle_session",
]
