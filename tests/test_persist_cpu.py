"""NEXT-1 persistence + restore on the host (-m "not gpu"): the C++ writer/loader of
libgockpt against the independent Python format oracle (oracle/ckpt_file.py), CRC corruption
detection, truncation, fault-injected crashes (atomic publication: LATEST never points at a
torn file), and the paper's "wait for the previous checkpoint" ordering at the ABI level."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import gockpt_inputs as gi
from oracle import ckpt_file as OF

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def G():
    from paper_2511_07035_b200 import build as gbuild
    gbuild.build()
    import paper_2511_07035_b200 as G
    return G


def state(n, seed=3):
    return [np.ascontiguousarray(x) for x in gi.warm_state(seed, n)]


@pytest.mark.parametrize("n", [1, 1000, (64 << 20) // 4 + 17, 3 * (64 << 20) // 4])   # 1..3 blocks + ragged
def test_cpp_writes_python_reads(G, tmp_path, n):
    p, m, v = state(n)
    path = str(tmp_path / "ck.bin")
    st = G.write_checkpoint(path, p, m, v, step=123, adam_t=120, rank=2, world=8, threads=4, meta_json='{"x": 1}')
    assert st["bytes"] == os.path.getsize(path) and st["gbs"] > 0
    hdr, rp, rm, rv = OF.read(path)
    assert hdr == dict(step=123, adam_t=120, n=n, rank=2, world=8, beta1=0.9, beta2=0.999, eps=1e-8,
                       weight_decay=0.01)
    for a, b in zip((rp, rm, rv), (p, m, v)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    meta = json.load(open(path + ".meta.json"))
    assert meta["step"] == 123 and meta["adam_t"] == 120 and meta["user"] == {"x": 1}
    assert OF.latest(str(tmp_path), 2) == path
    assert not os.path.exists(path + ".tmp")


@pytest.mark.parametrize("n", [5, (64 << 20) // 4 * 2 + 3])
def test_python_writes_cpp_reads(G, tmp_path, n):
    p, m, v = state(n, 9)
    path = str(tmp_path / "py.bin")
    OF.write(path, p, m, v, step=7, adam_t=7)
    assert G.read_header(path)["step"] == 7
    rp, rm, rv, hdr, st = G.load_checkpoint(path, n, threads=3)
    assert hdr["adam_t"] == 7 and hdr["n"] == n
    for a, b in zip((rp, rm, rv), (p, m, v)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_corruption_and_truncation_detected(G, tmp_path):
    from paper_2511_07035_b200 import GckError
    from paper_2511_07035_b200 import _lib as L
    n = (64 << 20) // 4 + 100
    p, m, v = state(n)
    path = str(tmp_path / "c.bin")
    G.write_checkpoint(path, p, m, v, step=1, adam_t=1)
    hdr = OF.read(path)[0]
    _, nblocks, table_off, table_bytes, offs, total = OF.layout(n)
    for where in (offs[0] + 5, offs[1] + (64 << 20) + 3, offs[2] + 4 * n - 1, table_off + 2, 40):
        bad = str(tmp_path / f"bad{where}.bin")
        data = bytearray(open(path, "rb").read())
        data[where] ^= 0x04                                      # one flipped bit
        open(bad, "wb").write(bytes(data))
        with pytest.raises(GckError) as e:
            G.load_checkpoint(bad, n)
        assert e.value.status == L.E_CORRUPT
        with pytest.raises(ValueError):
            OF.read(bad)
    trunc = str(tmp_path / "t.bin")
    open(trunc, "wb").write(open(path, "rb").read()[: offs[2] + 1000])
    with pytest.raises(GckError) as e:
        G.load_checkpoint(trunc, n)
    assert e.value.status == L.E_CORRUPT
    with pytest.raises(GckError) as e:
        G.load_checkpoint(path, n + 1)                           # wrong shard size
    assert e.value.status == L.E_INVALID
    with pytest.raises(GckError) as e:
        G.load_checkpoint(str(tmp_path / "missing.bin"), n)
    assert e.value.status == L.E_IO


def test_crash_during_persist_keeps_previous_latest(G, tmp_path):
    # SPEC S:370-373 persistence atomicity: a writer killed mid-way never publishes a torn file
    n = (64 << 20) // 4 * 2
    p, m, v = state(n)
    good = str(tmp_path / "ck_100.bin")
    G.write_checkpoint(good, p, m, v, step=100, adam_t=100)
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); import numpy as np, paper_2511_07035_b200 as G;"
            f"x = np.ones({n}, np.float32); G.write_checkpoint({str(tmp_path / 'ck_200.bin')!r}, x, x, x, "
            f"step=200, adam_t=200)")
    env = dict(os.environ, GCK_FAULT_PERSIST="2")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode != 0 and "GCK_E_ABORTED" in r.stderr
    assert OF.latest(str(tmp_path)) == good                      # LATEST still the previous checkpoint
    assert not os.path.exists(tmp_path / "ck_200.bin")           # never renamed into place
    hdr, rp, _, _ = OF.read(OF.latest(str(tmp_path)))
    assert hdr["step"] == 100 and np.array_equal(rp, p)
    # a process killed outright (SIGKILL) mid-write behaves the same
    big = (64 << 20) // 4 * 12
    code2 = (f"import sys; sys.path.insert(0, {ROOT!r}); import numpy as np, paper_2511_07035_b200 as G;"
             f"x = np.ones({big}, np.float32); print('go', flush=True); G.write_checkpoint("
             f"{str(tmp_path / 'ck_300.bin')!r}, x, x, x, step=300, adam_t=300, threads=1)")
    proc = subprocess.Popen([sys.executable, "-c", code2], stdout=subprocess.PIPE, text=True)
    assert proc.stdout.readline().strip() == "go"
    import time
    t_end = time.time() + 60
    while not os.path.exists(tmp_path / "ck_300.bin.tmp") and time.time() < t_end:
        time.sleep(0.001)                                # kill as soon as the writer has started
    proc.kill()
    proc.wait()
    assert OF.latest(str(tmp_path)) == good
    assert not os.path.exists(tmp_path / "ck_300.bin")


def test_range_loader(G, tmp_path):
    from paper_2511_07035_b200 import GckError
    from paper_2511_07035_b200 import _lib as L
    n = (64 << 20) // 4 * 2 + 12345                      # 3 blocks per section, ragged
    p, m, v = state(n, 5)
    path = str(tmp_path / "r.bin")
    G.write_checkpoint(path, p, m, v, step=9, adam_t=9)
    B = (64 << 20) // 4
    for off, cnt in [(0, 1), (B - 3, 7), (B, B), (5, 2 * B + 100), (n - 10, 10), (0, n), (n, 0)]:
        rp, rm, rv, h = G.load_checkpoint_range(path, off, cnt)
        assert h["step"] == 9
        for got, exp in zip((rp, rm, rv), (p, m, v)):
            assert np.array_equal(got.view(np.uint32), exp[off:off + cnt].view(np.uint32)), (off, cnt)
    with pytest.raises(GckError) as e:
        G.load_checkpoint_range(path, n - 5, 6)
    assert e.value.status == L.E_INVALID
    # corruption in a block the range touches is detected; in an untouched block it is not read
    _, nblocks, table_off, _, offs, _ = OF.layout(n)
    data = bytearray(open(path, "rb").read())
    data[offs[1] + 4 * (2 * B + 50)] ^= 1                  # m, block 2
    bad = str(tmp_path / "bad.bin")
    open(bad, "wb").write(bytes(data))
    with pytest.raises(GckError) as e:
        G.load_checkpoint_range(bad, 2 * B + 10, 100)
    assert e.value.status == L.E_CORRUPT
    rp, rm, rv, _ = G.load_checkpoint_range(bad, 0, B)        # blocks 0 only: fine
    assert np.array_equal(rm, m[:B])


# ---- NEXT-2 replay-on-restore: version-2 files (captured parts + gradient log + StepRecords) ----------

def _session_inputs(n, K, t0=10, seed=11, A=1024):
    """A seeded session from S(t0): the oracle's capture (parts at S(t0+i-1), glog, recs) and O1's S(T)."""
    import oracle
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(seed, n)
    grads = [gi.grad_bits(seed, t0 + i, n) for i in range(1, K + 1)]
    recs = [oracle.make_step_record(t=t0 + i, lr=1e-3 * (1 + 0.1 * i), **hp) for i in range(1, K + 1)]
    parts = oracle.make_parts(n, K, A)
    cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, recs, parts)
    want = oracle.trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]
    return oracle.assemble(cap), glog, recs, parts, want


def _crec(G, r):
    from paper_2511_07035_b200 import _lib as L
    return L.StepRecord(r.b1, r.c1, r.b2, r.c2, r.bc1, r.bc2, r.lr, r.eps, r.wd, r.gs, int(r.skip), 0, r.t)


def _eq(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


@pytest.mark.parametrize("n,K", [(5000, 1), (5000, 2), (70001, 4), ((64 << 20) // 2 + 777, 3)])
def test_log_file_cpp_writes_both_load_to_S_T(G, tmp_path, n, K):
    """C++ v2 writer -> (a) C++ loader replays on the host, (b) the Python format oracle + oracle
    replay: both == O1's S(T) bit for bit; the log header round-trips (plan, records, t0)."""
    (cp, cm, cv), glog, recs, parts, want = _session_inputs(n, K)
    path = str(tmp_path / "v2.bin")
    st = G.write_checkpoint_log(path, cp, cm, cv, t0=10, parts=parts, recs=[_crec(G, r) for r in recs],
                                glog=glog, adam_t=10 + K - 1, threads=3)
    assert st["bytes"] == os.path.getsize(path)
    h = G.read_header(path)
    assert h["version"] == (2) and h["step"] == 10 + K - 1
    lh = G.read_log_header(path)
    assert lh["t0"] == 10 and lh["K"] == K and lh["parts"] == [tuple(p) for p in parts]
    assert [r.t for r in lh["recs"]] == [r.t for r in recs]
    rp, rm, rv, hdr, _ = G.load_checkpoint(path, n, threads=4)
    for got, exp in zip((rp, rm, rv), want):
        assert _eq(got, exp)
    ohdr, op, om, ov = OF.read_consistent(path)
    assert ohdr["step"] == 10 + K - 1
    for got, exp in zip((op, om, ov), want):
        assert _eq(got, exp)
    # without the replay the captured bytes are what was written (and differ from S(T) for K > 1)
    _, sp, sm, sv = OF.read(path)
    assert _eq(sp, cp) and _eq(sm, cm) and _eq(sv, cv)
    if K > 1:
        assert not _eq(sp, want[0])


@pytest.mark.parametrize("n,K", [(4097, 2), (200003, 5)])
def test_log_file_python_writes_cpp_loads(G, tmp_path, n, K):
    (cp, cm, cv), glog, recs, parts, want = _session_inputs(n, K, seed=4)
    path = str(tmp_path / "py2.bin")
    OF.write_v2(path, cp, cm, cv, t0=10, parts=parts, recs=recs, glog=glog, adam_t=10 + K - 1)
    rp, rm, rv, hdr, _ = G.load_checkpoint(path, n, threads=2)
    assert hdr["step"] == 10 + K - 1
    for got, exp in zip((rp, rm, rv), want):
        assert _eq(got, exp)
    # the two writers produce the same bytes
    path2 = str(tmp_path / "c2.bin")
    G.write_checkpoint_log(path2, cp, cm, cv, t0=10, parts=parts, recs=[_crec(G, r) for r in recs], glog=glog,
                           adam_t=10 + K - 1, threads=2)
    assert open(path, "rb").read() == open(path2, "rb").read()


def test_log_file_range_loader_replays_the_range(G, tmp_path):
    """Resharded load of a v2 file: every range == the same range of S(T) (elementwise update)."""
    n, K = (64 << 20) // 2 + 4099, 4          # gradient slices span 2 blocks; state 1-2 blocks
    (cp, cm, cv), glog, recs, parts, want = _session_inputs(n, K, seed=8)
    path = str(tmp_path / "r2.bin")
    G.write_checkpoint_log(path, cp, cm, cv, t0=10, parts=parts, recs=[_crec(G, r) for r in recs], glog=glog,
                           adam_t=10 + K - 1)
    B = (64 << 20) // 2
    b1, b2 = parts[0][1], parts[1][1]
    for off, cnt in [(0, 1), (b1 - 5, 10), (b2 - 3, 7), (B - 2, 9), (parts[-1][0], n - parts[-1][0]), (0, n),
                     (n - 1, 1), (7, 0)]:
        rp, rm, rv, h = G.load_checkpoint_range(path, off, cnt, threads=2)
        for got, exp in zip((rp, rm, rv), want):
            assert _eq(got, exp[off:off + cnt]), (off, cnt)


def test_log_file_corruption_and_validation(G, tmp_path):
    from paper_2511_07035_b200 import GckError
    from paper_2511_07035_b200 import _lib as L
    n, K = 30000, 3
    (cp, cm, cv), glog, recs, parts, want = _session_inputs(n, K, seed=2)
    crecs = [_crec(G, r) for r in recs]
    path = str(tmp_path / "c.bin")
    G.write_checkpoint_log(path, cp, cm, cv, t0=10, parts=parts, recs=crecs, glog=glog, adam_t=12)
    log_off, table_off, _, _, slice_off, _ = OF._log_layout(n, K, parts)
    data = open(path, "rb").read()
    for where in (slice_off[1] + 3, log_off + 40, table_off + 1):   # gradient byte, log plan, CRC table
        bad = bytearray(data)
        bad[where] ^= 0x10
        bp = str(tmp_path / f"bad{where}.bin")
        open(bp, "wb").write(bytes(bad))
        with pytest.raises(GckError) as e:
            G.load_checkpoint(bp, n)
        assert e.value.status == L.E_CORRUPT
        with pytest.raises(ValueError):
            OF.read_consistent(bp)
    trunc = str(tmp_path / "t.bin")
    open(trunc, "wb").write(data[:slice_off[1] + 10])
    with pytest.raises(GckError) as e:
        G.load_checkpoint(trunc, n)
    assert e.value.status == L.E_CORRUPT
    # a version-1 file has no replay log
    v1 = str(tmp_path / "v1.bin")
    G.write_checkpoint(v1, cp, cm, cv, step=12, adam_t=12)
    with pytest.raises(GckError) as e:
        G.read_log_header(v1)
    assert e.value.status == L.E_INVALID
    # writer validation: a plan that does not cover [0, n), a non-contiguous one, K = 0
    bad_parts = [parts[0], (parts[1][0] + 1, parts[1][1]), parts[2]]
    for pp in (bad_parts, parts[:2]):
        with pytest.raises(GckError) as e:
            G.write_checkpoint_log(str(tmp_path / "x.bin"), cp, cm, cv, t0=10, parts=pp, recs=crecs, glog=glog,
                                   adam_t=12)
        assert e.value.status == L.E_INVALID


def test_log_file_with_skipped_update(G, tmp_path):
    """A skipped update inside the session (overflow step) is a no-op in the replay too."""
    import oracle
    n, K, t0, seed = 9000, 4, 20, 6
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(seed, n)
    grads = [gi.grad_bits(seed, t0 + i, n) for i in range(1, K + 1)]
    # update t0+2 skipped: bias-correction counts 21, (skip), 22, 23
    ts = [21, 21, 22, 23]
    recs = [oracle.make_step_record(t=ts[i], lr=1e-3, skip=(i == 1), **hp) for i in range(K)]
    parts = oracle.make_parts(n, K, 1024)
    cap, glog, _ = oracle.capture_session(p0, m0, v0, grads, recs, parts)
    want = oracle.trajectory(p0, m0, v0, grads[:K - 1], recs[:K - 1])[-1]
    cp, cm, cv = oracle.assemble(cap)
    path = str(tmp_path / "s.bin")
    G.write_checkpoint_log(path, cp, cm, cv, t0=t0, parts=parts, recs=[_crec(G, r) for r in recs], glog=glog,
                           adam_t=22)
    rp, rm, rv, _, _ = G.load_checkpoint(path, n)
    for got, exp in zip((rp, rm, rv), want):
        assert _eq(got, exp)
