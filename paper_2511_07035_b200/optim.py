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

import json
import os
import re

from ._lib import E_ABORTED, E_CORRUPT, E_INCOMPLETE, E_IO, GckError
from .gockpt import GoCkpt

# failures of the checkpoint path that void one checkpoint while training continues
_CKPT_FAILURES = (E_ABORTED, E_INCOMPLETE, E_CORRUPT, E_IO)
_FILE_RE = re.compile(r"^ckpt_(\d+)\.rank(\d+)\.bin$")


def resolve_restore_path(persist_dir: str, rank: int, world: int) -> str:
    """The file rank `rank` resumes from. With world > 1 it is the global checkpoint of MANIFEST.json
    (written by rank 0 only once every rank's shard was durable), so all ranks resume from the
    same step; a single rank uses its own LATEST.rank<r> pointer."""
    if world > 1:
        man_path = os.path.join(persist_dir, "MANIFEST.json")
        with open(man_path) as fh:
            man = json.load(fh)
        if man["world"] != world:
            raise ValueError(f"MANIFEST.json is for {man['world']} ranks, this job has {world}: "
                             "use harness.load_resharded")
        return os.path.join(persist_dir, man["files"][rank])
    with open(os.path.join(persist_dir, f"LATEST.rank{rank}")) as fh:
        return os.path.join(persist_dir, fh.read().strip())


def prune_checkpoints(persist_dir: str, rank: int, keep: int) -> list[str]:
    """Delete this rank's checkpoint files except the `keep` newest steps and the steps LATEST.rank<r>
    and MANIFEST.json point to (a crash while persisting must leave a loadable checkpoint). Also
    removes this rank's stale `.tmp` files of older steps. Returns the deleted paths."""
    if keep <= 0:
        return []
    steps = {}
    for f in os.listdir(persist_dir):
        mt = _FILE_RE.match(f)
        if mt and int(mt.group(2)) == rank:
            steps[int(mt.group(1))] = f
    protect = set(sorted(steps)[-keep:])
    for ptr in (f"LATEST.rank{rank}", "MANIFEST.json"):
        path = os.path.join(persist_dir, ptr)
        try:
            with open(path) as fh:
                text = fh.read()
        except OSError:
            continue
        names = json.loads(text)["files"] if ptr == "MANIFEST.json" else [text.strip()]
        for nm in names:
            mt = _FILE_RE.match(os.path.basename(nm))
            if mt:
                protect.add(int(mt.group(1)))
    gone = []
    newest = max(steps) if steps else -1
    for st, f in steps.items():
        if st in protect:
            continue
        for extra in ("", ".meta.json"):
            path = os.path.join(persist_dir, f + extra)
            if os.path.exists(path):
                os.unlink(path)
                gone.append(path)
    for f in os.listdir(persist_dir):  # partial files of older steps (a writer that died)
        if f.endswith(".tmp") and _FILE_RE.match(f[:-4]):
            mt = _FILE_RE.match(f[:-4])
            if int(mt.group(2)) == rank and int(mt.group(1)) < newest:
                os.unlink(os.path.join(persist_dir, f))
                gone.append(os.path.join(persist_dir, f))
    return gone


class CheckpointedAdamW:
    def __init__(self, master, exp_avg, exp_avg_sq, param_bf16=None, *, lr=1e-3, betas=(0.9, 0.999), eps=1e-8,
                 weight_decay=0.01, K=8, k_min=None, k_max=None, step=0, adam_t=None, persist_dir=None,
                 rank=0, world=1, on_checkpoint=None, keep=2, **ctx_kw):
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
        self._draining = None                         # (t0, K) of a finished session awaiting consistency
        self._persisting = False
        self._held = False                            # a finalized checkpoint not yet released
        self.last = None                              # (step, path or None) of the last consistent checkpoint
        self.keep = keep                              # checkpoints of this rank kept on disk (0 = all)
        self.failures = []                            # (step T, status name, message) of voided checkpoints
        self._commit = None                           # [T, durable] of a session awaiting the global commit
        if persist_dir:
            os.makedirs(persist_dir, exist_ok=True)

    # -- the paper's save_checkpoint hook
    def save_checkpoint(self):
        """Begin a checkpoint of the current state S(step) spread over the next K updates."""
        self._pending = True

    def _void(self, err: GckError):
        """A checkpoint-path failure (ABORTED / INCOMPLETE / CORRUPT): drop the session and keep
        training; the next save_checkpoint starts a fresh one."""
        t0, K = self._session if self._session is not None else self._draining
        self.failures.append((t0 + K - 1, str(err).split(":")[0], str(err)))
        if self.persist_dir:
            self._commit = [t0 + K - 1, False]  # the other ranks still expect this step's global commit
        self._session = None
        self._draining = None
        self._held = False
        self.ctx.release()  # ABORTED -> IDLE; waits until nothing of the session still lands

    def _settle(self, block: bool) -> bool:
        """Advance a finished session: consistent -> persist (background) -> released."""
        if self._draining is not None:
            try:
                ck = self.ctx.finalize(block=block)
            except GckError as e:
                if e.status not in _CKPT_FAILURES:
                    raise
                self._void(e)
                ck = None
            if ck is None:
                if self._draining is not None:
                    return False
            else:
                path = None
                if self.persist_dir:
                    path = os.path.join(self.persist_dir, f"ckpt_{ck.step}.rank{self.rank}.bin")
                    self.ctx.persist_begin(path, self.rank, self.world)
                    self._persisting = True
                    self._commit = [ck.step, False]
                self.last = (ck.step, path)
                if self.on_checkpoint:
                    self.on_checkpoint(ck)
                self._draining = None
                self._held = True
        if self._persisting:
            if not block:
                return False          # released once durable (gck_release waits for the persist)
            try:
                self.ctx.persist_wait()
                self._commit[1] = True
            except GckError as e:
                if e.status not in _CKPT_FAILURES:
                    raise
                self.failures.append((self.last[0], str(e).split(":")[0], str(e)))
                self.last = (self.last[0], None)
            self._persisting = False
        if self._held:
            self.ctx.release()
            self._held = False
        if block and self._commit is not None:
            self._global_commit()
        return True

    def _global_commit(self):
        """Every rank reaches this at the same global step (save_checkpoint / wait / close run in
        lock-step): publish MANIFEST.json when all shards of step T are durable, then prune."""
        step, ok = self._commit
        self._commit = None
        if self.world > 1:
            from .harness import commit_global
            ok = commit_global(self.persist_dir, step, ok,
                               files=[f"ckpt_{step}.rank{r}.bin" for r in range(self.world)])
        if ok and self.keep:
            prune_checkpoints(self.persist_dir, self.rank, self.keep)

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
        try:
            self.ctx.submit(part, self.global_step, max(self.adam_t, 1), self.lr if lr is None else lr, grad,
                            grad_scale, skip, stream)
        except GckError as e:  # the update still ran (as a plain step); only the checkpoint is void
            if e.status not in _CKPT_FAILURES or self._session is None:
                raise
            self._void(e)
            return
        if self._session is not None and part == self._session[1]:
            self._draining = self._session
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
        """Load a persisted checkpoint (path None: the global MANIFEST.json's file for this rank when
        world > 1, else this rank's LATEST) into the device
        state and resume after it: version-1 files upload S(T); version-2 (replay-on-restore)
        files are replayed on the GPU in place. Returns the file header."""
        if self._session is not None or self._draining is not None or self._held:
            raise RuntimeError("restore while a checkpoint session is live")
        if path is None:
            path = resolve_restore_path(self.persist_dir or ".", self.rank, self.world)
        h = self.ctx.restore(path, stream)
        self.global_step, self.adam_t = h["step"], h["adam_t"]
        return h

    def close(self):
        try:
            if self._session is None:
                self._settle(block=True)
        finally:
            self.ctx.close()
