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
