"""A training-loop face for the GoCkpt context: the paper's three hooks (§4.6:
"save_checkpoint, backward_begin, and update_begin") folded into an optimizer object.

    opt = CheckpointedAdamW(master, exp_avg, exp_avg_sq, param_bf16, lr=3e-4, K=8,
                            persist_dir="ckpts", rank=rank, world=world)
    for step in ...:
        loss.backward()                      # -> bf16 gradient shard `grad`
        if step % 100 == 0:
            opt.save_checkpoint()            # the next K updates carry the session
        opt.step(grad)                       # the fused AdamW step (+ pack) in libgockpt
    opt.wait()                               # last checkpoint consistent (and durable)

Host-side bookkeeping only (which part a step is, when to finalize / persist / release); every
update, pack, drain and replay runs in libgockpt. The session completes in the background:
`step()` polls `gck_finalize_poll` and, once the checkpoint is consistent, starts the
background persist and releases it when that finishes (the next `save_checkpoint` waits for
it).
"""

from __future__ import annotations

import os

from .gockpt import GoCkpt


class CheckpointedAdamW:
    def __init__(self, master, exp_avg, exp_avg_sq, param_bf16=None, *, lr=1e-3, betas=(0.9, 0.999), eps=1e-8,
                 weight_decay=0.01, K=8, k_min=None, k_max=None, step=0, adam_t=None, persist_dir=None,
                 rank=0, world=1, on_checkpoint=None, **ctx_kw):
        if ctx_kw.get("replay_mode") == "deferred" and not persist_dir:
            raise ValueError("replay_mode='deferred' materialises S(T) only when the file is loaded: "
                             "it needs persist_dir")
        self.K = K
        self.lr = lr
        self.ctx = GoCkpt(master, exp_avg, exp_avg_sq, param_bf16, beta1=betas[0], beta2=betas[1], eps=eps,
                          weight_decay=weight_decay, k_min=k_min or (1 if K == 0 else K),
                          k_max=k_max or (32 if K == 0 else K), **ctx_kw)
        self.global_step = step                       # training-step index of the last update
        self.adam_t = step if adam_t is None else adam_t
        self.persist_dir = persist_dir
        self.rank, self.world = rank, world
        self.on_checkpoint = on_checkpoint
        self._pending = False                         # save_checkpoint() requested
        self._session = None                          # (t0, K) while parts are being submitted
        self._draining = None                         # t0 of a finished session awaiting consistency
        self._persisting = False
        self._held = False                            # a finalized checkpoint not yet released
        self.last = None                              # (step, path or None) of the last consistent checkpoint
        if persist_dir:
            os.makedirs(persist_dir, exist_ok=True)

    # -- the paper's save_checkpoint hook
    def save_checkpoint(self):
        """Begin a checkpoint of the current state S(step) spread over the next K updates."""
        self._pending = True

    def _settle(self, block: bool) -> bool:
        """Advance a finished session: consistent -> persist (background) -> released."""
        if self._draining is not None:
            ck = self.ctx.finalize(block=block)
            if ck is None:
                return False
            path = None
            if self.persist_dir:
                path = os.path.join(self.persist_dir, f"ckpt_{ck.step}.rank{self.rank}.bin")
                self.ctx.persist_begin(path, self.rank, self.world)
                self._persisting = True
            self.last = (ck.step, path)
            if self.on_checkpoint:
                self.on_checkpoint(ck)
            self._draining = None
            self._held = True
        if self._persisting:
            if not block:
                return False          # released once durable (gck_release waits for the persist)
            self.ctx.persist_wait()
            self._persisting = False
        if self._held:
            self.ctx.release()
            self._held = False
        return True

    # -- the update (the paper's update_begin hook is this call)
    def step(self, grad, lr=None, grad_scale=1.0, skip=False, stream=None):
        if self._draining is not None:
            self._settle(block=False)
        part = 0
        if self._session is None and self._pending:
            self._settle(block=True)                  # the previous checkpoint must be done
            self.ctx.begin_checkpoint(self.global_step, self.K)
            K = self.ctx.stats()["last_session_k"]
            self._session = (self.global_step, K)
            self._pending = False
        self.global_step += 1
        if not skip:
            self.adam_t += 1
        if self._session is not None:
            t0, K = self._session
            part = self.global_step - t0
        self.ctx.submit(part, self.global_step, max(self.adam_t, 1), self.lr if lr is None else lr, grad,
                        grad_scale, skip, stream)
        if self._session is not None and part == self._session[1]:
            self._draining = self._session[0]
            self._session = None

    def grad_fence(self, stream=None):
        """Direct staging: call before the next backward overwrites the gradient buffer."""
        self.ctx.grad_fence(stream)

    def wait(self) -> tuple | None:
        """Block until the last requested checkpoint is consistent (and durable); returns (step, path)."""
        if self._session is not None:
            raise RuntimeError("a session is still collecting parts: run K more steps first")
        self._settle(block=True)
        return self.last

    def restore(self, path: str | None = None, stream=None) -> dict:
        """Load a persisted checkpoint (the LATEST of this rank if path is None) into the device
        state and resume after it: version-1 files upload S(T); version-2 (replay-on-restore)
        files are replayed on the GPU in place. Returns the file header."""
        if self._session is not None or self._draining is not None or self._held:
            raise RuntimeError("restore while a checkpoint session is live")
        if path is None:
            latest = os.path.join(self.persist_dir or ".", f"LATEST.rank{self.rank}")
            with open(latest) as fh:
                path = os.path.join(os.path.dirname(latest), fh.read().strip())
        h = self.ctx.restore(path, stream)
        self.global_step, self.adam_t = h["step"], h["adam_t"]
        return h

    def close(self):
        try:
            if self._session is None:
                self._settle(block=True)
        finally:
            self.ctx.close()
