"""World-size-2 gloo tests of the N>1 host logic (-m "not gpu").

The checkpoint path shards with no exchange step (§4.5: each data-parallel rank saves
its own optimizer shard): every rank plans its own K parts over its own ZeRO-1 shard, derives
the same session schedule from the global step, and the global checkpoint is the
concatenation of the per-rank ones. Timings are maxed over ranks; the global commit is an
all-ranks-finalized MIN reduction ("Rank 0 monitoring completion by other Ranks").
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gockpt_inputs as gi
import oracle

HP = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, K, t0, result_dir, deferred=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_07035_b200 import build as gbuild
        gbuild.build()
        import paper_2511_07035_b200 as G
        from paper_2511_07035_b200.harness import zero1_shard, max_over_ranks, all_ranks_ok, session_part

        off, n_r, padded = zero1_shard(n_total, world, rank, align=64)
        # identical schedule on every rank, derived from the global step only
        sched = [session_part(j, K) for j in range(0, 12)]
        gathered = [None] * world
        dist.all_gather_object(gathered, sched)
        assert all(g == sched for g in gathered)
        # this rank's shard: its state and gradients are the global vector's [off, off+n_r)
        idx = np.arange(off, off + n_r, dtype=np.uint64)
        p0, m0, v0 = gi.warm_state(42, idx)
        grads = [gi.grad_bits(42, t0 + i, idx) for i in range(1, K + 1)]
        recs = [oracle.make_step_record(t=t0 + i, lr=1e-3, **HP) for i in range(1, K + 1)]
        parts = G.plan_parts(n_r, K, 64)
        cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, recs, parts)
        p, m, v = (np.ascontiguousarray(x) for x in oracle.assemble(cap))
        lrecs = [G.make_step_record(0.9, 0.999, 1e-8, 0.01, t0 + i, 1e-3) for i in range(1, K + 1)]
        cp, cm, cv = p.copy(), m.copy(), v.copy()           # the captured parts (replay-on-restore file)
        G.replay_host(lrecs, parts, p, m, v, [np.ascontiguousarray(x) for x in glog], threads=2)
        np.save(os.path.join(result_dir, f"rank{rank}.npy"), np.stack([p, m, v]))
        # NEXT-1 per-rank persistence + rank-0 global commit
        from paper_2511_07035_b200.harness import commit_global
        path = os.path.join(result_dir, f"ckpt_{t0 + K - 1}.rank{rank}.bin")
        if deferred:      # version 2: captured parts + gradient log; every loader replays
            G.write_checkpoint_log(path, cp, cm, cv, t0=t0, parts=parts, recs=lrecs,
                                   glog=[np.ascontiguousarray(x) for x in glog], adam_t=t0 + K - 1, rank=rank,
                                   world=world, threads=2)
        else:
            G.write_checkpoint(path, p, m, v, step=t0 + K - 1, adam_t=t0 + K - 1, rank=rank, world=world, threads=2)
        assert commit_global(result_dir, t0 + K - 1, True, n_total=n_total, n_per_rank=n_r, align=64)
        t = max_over_ranks(float(rank + 1))
        assert t == float(world)
        assert all_ranks_ok(True)
        ok = all_ranks_ok(rank != 1)          # one rank failing voids the global checkpoint
        assert ok is False
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total,deferred", [(10_000, False), (4096 * 3 + 17, False), (4096 * 3 + 17, True)])
def test_two_ranks_shard_checkpoints_concatenate_to_global(tmp_path, n_total, deferred):
    world, K, t0 = 2, 4, 20
    mp.spawn(_worker, args=(world, _free_port(), n_total, K, t0, str(tmp_path), deferred), nprocs=world, join=True)
    from paper_2511_07035_b200.harness import zero1_shard
    _, n_r, padded = zero1_shard(n_total, world, 0, align=64)
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)], axis=1)
    idx = np.arange(padded, dtype=np.uint64)
    p0, m0, v0 = gi.warm_state(42, idx)
    grads = [gi.grad_bits(42, t0 + i, idx) for i in range(1, K)]
    recs = [oracle.make_step_record(t=t0 + i, lr=1e-3, **HP) for i in range(1, K)]
    want = oracle.trajectory(p0, m0, v0, grads, recs)[-1]
    for g, w in zip(got, want):
        assert np.array_equal(g.view(np.uint32), w.view(np.uint32))
    # the global manifest names every rank's durable file; reading them back gives S(T) again
    import json
    from oracle import ckpt_file as OF
    man = json.load(open(tmp_path / "MANIFEST.json"))
    assert man["step"] == t0 + K - 1 and man["world"] == world
    back = np.concatenate([np.stack(OF.read_consistent(str(tmp_path / f))[1:]) for f in man["files"]], axis=1)
    assert np.array_equal(back.view(np.uint32), got.view(np.uint32))
    # load into other data-parallel degrees (resharding): the concatenation over the new ranks is S(T)
    from paper_2511_07035_b200.harness import load_resharded
    for w_new in (1, 3, 4):
        parts = [load_resharded(str(tmp_path), w_new, r, align=64) for r in range(w_new)]
        assert all(p[3] == t0 + K - 1 for p in parts)
        cat = [np.concatenate([p[k] for p in parts])[:n_total] for k in range(3)]
        for c, w in zip(cat, want):
            assert np.array_equal(c.view(np.uint32), w[:n_total].view(np.uint32))
        pad = np.concatenate([p[0] for p in parts])[n_total:]
        assert not pad.any()                                     # ZeRO padding loads as zeros


def test_zero1_shard_layout():
    from paper_2511_07035_b200.harness import zero1_shard
    for n_total, world in [(124_439_808, 8), (6_738_415_616, 8), (13_015_864_320, 2), (1, 4)]:
        spans = [zero1_shard(n_total, world, r) for r in range(world)]
        padded = spans[0][2]
        assert padded >= n_total and padded % (world * 1024) == 0
        assert [s[0] for s in spans] == [r * spans[0][1] for r in range(world)]
        assert sum(s[1] for s in spans) == padded
    # Llama-2 7B over 8 ranks -> 842,301,952 per rank
    assert zero1_shard(6_738_415_616, 8, 0, align=512)[1] == 842_301_952
