"""NEXT-1 oracle: a plain Python reader/writer of the checkpoint file format
(TEST INFRASTRUCTURE ONLY; see oracle/__init__.py). Written from the format description in
include/gockpt.h (gck_file_header) — shares no code with persist.cpp — so files written by
either side must be readable, CRC-verified and value-identical on the other.

Paper anchors: P:359, P:367 (§4.4.1, §4.4.3: multi-threaded persistence, metadata written
last marks completion), P:352 (§4.3.2: load SSD -> CPU -> GPU, resume after the checkpoint).
CRC: CRC-32 with the zlib polynomial (zlib.crc32), per 64 MiB block of each section.
"""

from __future__ import annotations

import os
import struct
import zlib

import numpy as np

MAGIC = b"GOCKPT\x00\x01"
VERSION = 1
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


def read(path):
    """-> (header dict, master, m, v); raises ValueError on any format or CRC violation."""
    with open(path, "rb") as fh:
        raw = fh.read(PAGE)
        if len(raw) < HDR.size:
            raise ValueError("truncated header")
        f = HDR.unpack(raw[:HDR.size])
        (magic, version, hbytes, step, adam_t, n, rank, world, b1, b2, eps, wd, block, nblocks, table_off,
         o0, o1, o2, s0, s1, s2, table_crc, header_crc) = f
        if magic != MAGIC or version != VERSION:
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
    return hdr, out[0], out[1], out[2]


def latest(directory, rank=0):
    """The file the LATEST pointer of `rank` names, or None."""
    p = os.path.join(directory, f"LATEST.rank{rank}")
    if not os.path.exists(p):
        return None
    return os.path.join(directory, open(p).read().strip())
