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
