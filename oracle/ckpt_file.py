"""NEXT-1 oracle: a plain Python reader/writer of the checkpoint file format
(TEST INFRASTRUCTURE ONLY; see oracle/__init__.py). Written from the format description in
include/gockpt.h (gck_file_header) — shares no code with persist.cpp — so files written by
either side must be readable, CRC-verified and value-identical on the other.

Paper anchors: P:359, P:367 (§4.4.1, §4.4.3: multi-threaded persistence, metadata written
last marks completion), P:352 (§4.3.2: load SSD -> CPU -> GPU, resume after the checkpoint).
CRC: CRC-32 with the zlib polynomial (zlib.crc32), per 64 MiB block of each section.

Version 2 (replay-on-restore; gck_log_header in include/gockpt.h): the
sections hold the CAPTURED parts (part i at S(t0+i-1), §4.2.1), followed by the replay
log (plan, K StepRecords, gradient slices G(t0+i)[0:hi_i]); `read_consistent` applies the
oracle's own replay (oracle/replay.py, §4.3.1) to obtain S(T).
"""

from __future__ import annotations

import os
import struct
import zlib

import numpy as np

MAGIC = b"GOCKPT\x00\x01"
VERSION = 1
VERSION_LOG = 2
LOG_MAGIC = b"GCKRLOG\x00"
LOG_HEADER_BYTES = 8192
K_LIMIT = 64
# gck_step_record: b1 c1 b2 c2 bc1 bc2 lr eps wd gs (binary32), skip (int32), _pad, t (uint64)
REC = struct.Struct("<10fiIQ")
# gck_log_header: magic, K, _pad, t0, lo[64], hi[64], rec[64], glog_offset[64], glog_table_offset,
# glog_nblocks, glog_table_crc, log_crc
LOG_HEAD = struct.Struct(f"<8sIIQ{K_LIMIT}Q{K_LIMIT}Q")
LOG_TAIL = struct.Struct(f"<{K_LIMIT}QQQII")
PAGE = 4096
BLOCK = 64 << 20
# magic, version, header_bytes, step, adam_t, n, rank, world, beta1, beta2, eps, wd,
# block_bytes, nblocks, table_offset, section_offset[3], section_bytes[3], table_crc, header_crc
HDR = struct.Struct("<8sIIQQQIIddddQQQ3Q3QII")


def _align(x, a):
    return (x + a - 1) // a * a


def layout(n):
    sec = n * 4
    nblocks = (sec + BLOCK - 1) // BLOCK
    table_off = PAGE
    table_bytes = _align(3 * nblocks * 4, PAGE)
    offs, off = [], table_off + table_bytes
    for _ in range(3):
        offs.append(off)
        off = _align(off + sec, PAGE)
    return sec, nblocks, table_off, table_bytes, offs, off


def write(path, master, m, v, step, adam_t, rank=0, world=1, hp=(0.9, 0.999, 1e-8, 0.01)):
    n = len(master)
    sec, nblocks, table_off, table_bytes, offs, total = layout(n)
    secs = [np.ascontiguousarray(x, np.float32).tobytes() for x in (master, m, v)]
    table = [zlib.crc32(s[b * BLOCK:(b + 1) * BLOCK]) for s in secs for b in range(nblocks)]
    tbl = struct.pack(f"<{len(table)}I", *table)
    fields = [MAGIC, VERSION, PAGE, step, adam_t, n, rank, world, *hp, BLOCK, nblocks, table_off, *offs, *[sec] * 3,
              zlib.crc32(tbl), 0]
    raw = HDR.pack(*fields)
    fields[-1] = zlib.crc32(raw[:HDR.size - 4])
    raw = HDR.pack(*fields)
    with open(path, "wb") as fh:
        fh.truncate(total)
        fh.write(raw.ljust(PAGE, b"\0"))
        fh.seek(table_off)
        fh.write(tbl)
        for s, o in zip(secs, offs):
            fh.seek(o)
            fh.write(s)


def _log_layout(n, K, parts):
    """Offsets of the version-2 replay log: (log_off, table_off, table_bytes, nblocks, slice_off, end)."""
    log_off = layout(n)[5]
    table_off = log_off + LOG_HEADER_BYTES
    sizes = [parts[i][1] * 2 for i in range(K - 1)]
    nblocks = sum((b + BLOCK - 1) // BLOCK for b in sizes)
    table_bytes = _align(nblocks * 4, PAGE)
    off, slice_off = table_off + table_bytes, []
    for b in sizes:
        slice_off.append(off)
        off = _align(off + b, PAGE)
    return log_off, table_off, table_bytes, nblocks, slice_off, off


def _pack_rec(r):
    return REC.pack(float(r.b1), float(r.c1), float(r.b2), float(r.c2), float(r.bc1), float(r.bc2), float(r.lr),
                    float(r.eps), float(r.wd), float(r.gs), int(bool(r.skip)), 0, int(r.t))


def _unpack_rec(raw):
    from .adamw import StepRecord
    b1, c1, b2, c2, bc1, bc2, lr, eps, wd, gs, skip, _pad, t = REC.unpack(raw)
    f = np.float32
    return StepRecord(t=t, skip=bool(skip), b1=f(b1), c1=f(c1), b2=f(b2), c2=f(c2), bc1=f(bc1), bc2=f(bc2), lr=f(lr),
                      eps=f(eps), wd=f(wd), gs=f(gs))


def _log_bytes(K, t0, parts, recs, slice_off, table_off, nblocks, table_crc):
    lo = [parts[i][0] if i < K else 0 for i in range(K_LIMIT)]
    hi = [parts[i][1] if i < K else 0 for i in range(K_LIMIT)]
    body = LOG_HEAD.pack(LOG_MAGIC, K, 0, t0, *lo, *hi)
    body += b"".join(_pack_rec(recs[i]) if i < K else bytes(REC.size) for i in range(K_LIMIT))
    goff = [slice_off[i] if i < K - 1 else 0 for i in range(K_LIMIT)]
    tail = LOG_TAIL.pack(*goff, table_off, nblocks, table_crc, 0)
    raw = body + tail
    crc = zlib.crc32(raw[:-4])
    return raw[:-4] + struct.pack("<I", crc)


def write_v2(path, master, m, v, *, t0, parts, recs, glog, adam_t, rank=0, world=1, hp=(0.9, 0.999, 1e-8, 0.01)):
    """Version-2 file: master/m/v = the captured parts, parts = the K (lo, hi), recs[i-1] = StepRecord of update
    t0+i, glog[i-1] = G(t0+i)[0:hi_i] as uint16 (i < K)."""
    K, n = len(parts), len(master)
    write(path, master, m, v, step=t0 + K - 1, adam_t=adam_t, rank=rank, world=world, hp=hp)
    raw = bytearray(open(path, "rb").read())
    log_off, table_off, table_bytes, nblocks, slice_off, end = _log_layout(n, K, parts)
    slices = [np.ascontiguousarray(glog[i], np.uint16).tobytes() for i in range(K - 1)]
    table = [zlib.crc32(sb[b * BLOCK:(b + 1) * BLOCK]) for sb in slices for b in range((len(sb) + BLOCK - 1) // BLOCK)]
    tbl = struct.pack(f"<{len(table)}I", *table)
    raw.extend(bytes(end - len(raw)))
    raw[log_off:log_off + LOG_HEAD.size + K_LIMIT * REC.size + LOG_TAIL.size] = _log_bytes(
        K, t0, parts, recs, slice_off, table_off, nblocks, zlib.crc32(tbl))
    raw[table_off:table_off + len(tbl)] = tbl
    for sb, o in zip(slices, slice_off):
        raw[o:o + len(sb)] = sb
    f = list(HDR.unpack(bytes(raw[:HDR.size])))
    f[1] = VERSION_LOG
    f[-1] = 0
    h = HDR.pack(*f)
    f[-1] = zlib.crc32(h[:HDR.size - 4])
    raw[:HDR.size] = HDR.pack(*f)
    open(path, "wb").write(bytes(raw))


def read_log(path, n):
    """The replay log of a version-2 file -> dict(t0, K, parts, recs, glog); ValueError on any violation."""
    log_off = layout(n)[5]
    with open(path, "rb") as fh:
        fh.seek(log_off)
        raw = fh.read(LOG_HEAD.size + K_LIMIT * REC.size + LOG_TAIL.size)
        if len(raw) != LOG_HEAD.size + K_LIMIT * REC.size + LOG_TAIL.size:
            raise ValueError("truncated replay log header")
        head = LOG_HEAD.unpack(raw[:LOG_HEAD.size])
        magic, K, _pad, t0 = head[:4]
        lo, hi = head[4:4 + K_LIMIT], head[4 + K_LIMIT:4 + 2 * K_LIMIT]
        if magic != LOG_MAGIC:
            raise ValueError("replay log magic")
        if zlib.crc32(raw[:-4]) != struct.unpack("<I", raw[-4:])[0]:
            raise ValueError("replay log CRC mismatch")
        if not 1 <= K <= K_LIMIT:
            raise ValueError("replay log K")
        parts = [(lo[i], hi[i]) for i in range(K)]
        if parts[0][0] != 0 or parts[-1][1] != n or any(parts[i][1] != parts[i + 1][0] for i in range(K - 1)) \
                or any(a >= b for a, b in parts):
            raise ValueError("replay log plan")
        r0 = LOG_HEAD.size
        recs = [_unpack_rec(raw[r0 + i * REC.size:r0 + (i + 1) * REC.size]) for i in range(K)]
        tail = LOG_TAIL.unpack(raw[r0 + K_LIMIT * REC.size:])
        goff, table_off, nblocks, table_crc = tail[:K_LIMIT], tail[K_LIMIT], tail[K_LIMIT + 1], tail[K_LIMIT + 2]
        exp = _log_layout(n, K, parts)
        if (table_off, nblocks) != (exp[1], exp[3]) or list(goff[:K - 1]) != exp[4]:
            raise ValueError("replay log layout")
        fh.seek(table_off)
        tbl = fh.read(nblocks * 4)
        if zlib.crc32(tbl) != table_crc:
            raise ValueError("gradient CRC table mismatch")
        table = struct.unpack(f"<{nblocks}I", tbl)
        glog, k = [], 0
        for i in range(K - 1):
            fh.seek(goff[i])
            data = fh.read(parts[i][1] * 2)
            if len(data) != parts[i][1] * 2:
                raise ValueError("truncated gradient slice")
            for b in range((len(data) + BLOCK - 1) // BLOCK):
                if zlib.crc32(data[b * BLOCK:(b + 1) * BLOCK]) != table[k]:
                    raise ValueError(f"gradient CRC mismatch slice {i} block {b}")
                k += 1
            glog.append(np.frombuffer(data, np.uint16).copy())
    return dict(t0=t0, K=K, parts=parts, recs=recs, glog=glog)


def read_consistent(path):
    """-> (header dict, master, m, v) at S(T): a version-1 file as is; a version-2 file replayed with the
    oracle's own O2 replay (oracle/replay.py)."""
    from .replay import replay
    hdr, p, m, v = read(path)
    if hdr.get("version", VERSION) == VERSION:
        return hdr, p, m, v
    log = read_log(path, hdr["n"])
    if log["t0"] + log["K"] - 1 != hdr["step"]:
        raise ValueError("replay log t0 + K - 1 != header step")
    cap = [(p[a:b], m[a:b], v[a:b]) for a, b in log["parts"]]
    rp, rm, rv = replay(cap, log["glog"], log["recs"], log["parts"])
    return hdr, rp, rm, rv


def read(path):
    """-> (header dict, master, m, v); raises ValueError on any format or CRC violation."""
    with open(path, "rb") as fh:
        raw = fh.read(PAGE)
        if len(raw) < HDR.size:
            raise ValueError("truncated header")
        f = HDR.unpack(raw[:HDR.size])
        (magic, version, hbytes, step, adam_t, n, rank, world, b1, b2, eps, wd, block, nblocks, table_off,
         o0, o1, o2, s0, s1, s2, table_crc, header_crc) = f
        if magic != MAGIC or version not in (VERSION, VERSION_LOG):
            raise ValueError("bad magic/version")
        if zlib.crc32(raw[:HDR.size - 4]) != header_crc:
            raise ValueError("header CRC mismatch")
        fh.seek(table_off)
        tbl = fh.read(3 * nblocks * 4)
        if zlib.crc32(tbl) != table_crc:
            raise ValueError("table CRC mismatch")
        table = struct.unpack(f"<{3 * nblocks}I", tbl)
        out = []
        for k, (o, sb) in enumerate(((o0, s0), (o1, s1), (o2, s2))):
            fh.seek(o)
            data = fh.read(sb)
            if len(data) != sb:
                raise ValueError("truncated section")
            for b in range(nblocks):
                if zlib.crc32(data[b * block:(b + 1) * block]) != table[k * nblocks + b]:
                    raise ValueError(f"data CRC mismatch section {k} block {b}")
            out.append(np.frombuffer(data, np.float32).copy())
    hdr = dict(step=step, adam_t=adam_t, n=n, rank=rank, world=world, beta1=b1, beta2=b2, eps=eps, weight_decay=wd)
    if version != VERSION:
        hdr["version"] = version
    return hdr, out[0], out[1], out[2]


def latest(directory, rank=0):
    """The file the LATEST pointer of `rank` names, or None."""
    p = os.path.join(directory, f"LATEST.rank{rank}")
    if not os.path.exists(p):
        return None
    return os.path.join(directory, open(p).read().strip())
