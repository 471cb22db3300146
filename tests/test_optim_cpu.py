"""Host-side file logic of the optimizer face (-m "not gpu"): which file a rank resumes from and
which checkpoint files retention may delete (no GPU: plain files in a temp directory)."""

import json
import os

import pytest

from paper_2511_07035_b200.optim import prune_checkpoints, resolve_restore_path


def _touch(d, name, text="x"):
    with open(os.path.join(d, name), "w") as fh:
        fh.write(text)


def test_restore_path_single_rank_uses_latest(tmp_path):
    d = str(tmp_path)
    _touch(d, "LATEST.rank0", "ckpt_15.rank0.bin\n")
    assert resolve_restore_path(d, 0, 1) == os.path.join(d, "ckpt_15.rank0.bin")


def test_restore_path_multi_rank_uses_manifest_not_latest(tmp_path):
    """Rank 1 persisted step 27 but rank 0 crashed before its shard of 27 was durable: the manifest
    still says 15, and both ranks must resume from 15 (their LATEST files disagree)."""
    d = str(tmp_path)
    _touch(d, "LATEST.rank0", "ckpt_15.rank0.bin\n")
    _touch(d, "LATEST.rank1", "ckpt_27.rank1.bin\n")
    _touch(d, "MANIFEST.json", json.dumps({"step": 15, "world": 2, "files": ["ckpt_15.rank0.bin", "ckpt_15.rank1.bin"]}))
    assert resolve_restore_path(d, 0, 2) == os.path.join(d, "ckpt_15.rank0.bin")
    assert resolve_restore_path(d, 1, 2) == os.path.join(d, "ckpt_15.rank1.bin")
    with pytest.raises(ValueError):
        resolve_restore_path(d, 0, 4)


def test_prune_keeps_newest_and_pointed_to(tmp_path):
    d = str(tmp_path)
    for st in (3, 15, 27, 39, 51):
        for r in (0, 1):
            _touch(d, f"ckpt_{st}.rank{r}.bin")
            _touch(d, f"ckpt_{st}.rank{r}.bin.meta.json")
    _touch(d, "ckpt_63.rank0.bin.tmp")        # a newer write in flight: never touched
    _touch(d, "ckpt_27.rank0.bin.tmp")        # a dead writer's leftover of an older step
    _touch(d, "LATEST.rank0", "ckpt_51.rank0.bin\n")
    _touch(d, "MANIFEST.json", json.dumps({"step": 15, "world": 2, "files": ["ckpt_15.rank0.bin", "ckpt_15.rank1.bin"]}))
    gone = prune_checkpoints(d, 0, keep=2)
    left = sorted(os.listdir(d))
    for st in (15, 39, 51):                   # 2 newest + the manifest's step
        assert f"ckpt_{st}.rank0.bin" in left and f"ckpt_{st}.rank0.bin.meta.json" in left
    for st in (3, 27):
        assert f"ckpt_{st}.rank0.bin" not in left and f"ckpt_{st}.rank0.bin.meta.json" not in left
    assert "ckpt_63.rank0.bin.tmp" in left and "ckpt_27.rank0.bin.tmp" not in left
    assert all(f"ckpt_{st}.rank1.bin" in left for st in (3, 15, 27, 39, 51))   # other ranks' files untouched
    assert len(gone) == 5
    assert prune_checkpoints(d, 0, keep=0) == []


# ---------------------------------------------------------------- the optimizer face at world 2 (gloo)
class _FakeCtx:
    """Stands in for GoCkpt (no GPU here): records the calls, 'persists' a small file, and can void a
    chosen session the way the library does (finalize raises GCK_E_CORRUPT)."""

    def __init__(self, *a, fail_t=None, rank=0, **kw):
        self.fail_t, self.rank, self.sess, self.held = fail_t, rank, None, None

    def begin_checkpoint(self, t0, K):
        self.sess = (t0, K)

    def stats(self):
        return {"last_session_k": self.sess[1] if self.sess else 0}

    def submit(self, part, step, adam_t, lr, grad, gs=1.0, skip=False, stream=None):
        return 0

    def finalize(self, block=True):
        from paper_2511_07035_b200._lib import E_CORRUPT, GckError
        t0, K = self.sess
        if t0 + K - 1 == self.fail_t:
            raise GckError(E_CORRUPT, "drain verification: injected")
        from types import SimpleNamespace
        self.held = t0 + K - 1
        return SimpleNamespace(step=t0 + K - 1)

    def persist_begin(self, path, rank, world, meta_json=None):
        with open(path, "w") as fh:
            fh.write("x")
        d = os.path.dirname(path)
        with open(os.path.join(d, f"LATEST.rank{rank}"), "w") as fh:
            fh.write(os.path.basename(path) + "\n")

    def persist_wait(self):
        return {}

    def release(self):
        self.held = None

    def close(self):
        pass


def _opt_worker(rank, world, port, d, fail_rank, fail_t, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_07035_b200.optim as O
        O.GoCkpt = lambda *a, **kw: _FakeCtx(fail_t=fail_t if rank == fail_rank else None, rank=rank)
        opt = O.CheckpointedAdamW(None, None, None, K=4, persist_dir=d, rank=rank, world=world, keep=2)
        manifests = []
        for s in range(1, 61):
            if s % 12 == 1:
                opt.save_checkpoint()
            opt.step(None)
            if s % 12 == 1 and rank == 0 and os.path.exists(os.path.join(d, "MANIFEST.json")):
                manifests.append(json.load(open(os.path.join(d, "MANIFEST.json")))["step"])
        opt.wait()
        if rank == 0:
            manifests.append(json.load(open(os.path.join(d, "MANIFEST.json")))["step"])
        q.put((rank, [f[:2] for f in opt.failures], manifests, sorted(os.listdir(d))))
    finally:
        dist.destroy_process_group()


def test_global_manifest_lockstep_with_a_voided_rank(tmp_path):
    """world 2: checkpoints at T = 3, 15, 27, 39, 51; rank 1's T = 27 is voided (CORRUPT). Both ranks
    reach the global commit at the same steps (no deadlock), the manifest never names 27, it names
    the newest step every rank made durable, and retention keeps 2 files per rank plus the manifest's."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_opt_worker, args=(r, 2, port, str(tmp_path), 1, 27, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    res = dict((r, (f, m, ls)) for r, f, m, ls in (q.get(timeout=120) for _ in procs))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert res[0][0] == [] and res[1][0] == [(27, "GCK_E_CORRUPT")]
    manifests = res[0][1]
    assert 27 not in manifests and manifests[-1] == 51
    assert manifests == sorted(manifests)
    files = res[0][2]
    assert "ckpt_51.rank0.bin" in files and "ckpt_51.rank1.bin" in files and "ckpt_3.rank0.bin" not in files
