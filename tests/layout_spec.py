"""The library's DEVICE blob layout, written out from DESIGN.md section 4
("Blob layout") as a test specification (test infrastructure, not oracle).

The oracle reads and writes only the canonical row-major blob (SURVEY.md 8(b),
oracle/formats.py).  The library streams a tile-major layout instead and
converts canonical blobs with hb_repack_canonical; the GPU tests compare that
conversion with `device_blob` below byte for byte, and tests/test_layout_spec.py
pins these formulas with bytes worked out by hand.

Rows come in TILES of 16 rows; along K a row is cut into GROUPS of EPG
elements that occupy 64 bytes (EPG = 32 F16, 64 Q8, 128 Q4, 256 Q2; G = K/EPG
groups per row).  A UNIT = (tile, group) = the 16 rows' 64-byte pieces of that
group, stored contiguously (1 KB), units in (tile, group) order:

    code byte of element (n, k) = 1024*(G*tile + grp) + 64*r + o(k % EPG)
        tile = n // 16, r = n % 16, grp = k // EPG

with the within-group offset o (t = (k%32)//8, q = k%8, j = block in group):
    F16: o = 2*(k%32)
    Q8 : byte 16*t + 8*j + q                                (whole byte, int8)
    Q4 : byte 16*t + 4*j + q//2, bits 4*(q%2)..+3
    Q2 : byte 16*t + 4*(j//2) + 2*(q//4) + (j%2), bits 2*(q%4)..+1

Scales: one SB-byte record per (unit, row) -- SB = 2*BPG (d of the BPG blocks
of the group, fp16) and, for Q2, another 2*BPG bytes of m:

    scale record of (n, grp) at 16*SB*(G*tile + grp) + SB*r
        d of block j at +2*j,  m of block j at +2*BPG + 2*j   (Q2)

Q2K (R32): the codes as Q2; the 20-byte record of (n, grp) (one
super-block of 256) holds d (fp16) at +0, dmin (fp16) at +2 and the 16
sub-block bytes sc_j at +4 + j; the blob is padded to the canonical size.

Per matrix (W1, W3, W2): a code section then (quantised) one scale section,
each 256-byte aligned.  The total size equals the canonical blob's.
"""
from __future__ import annotations

import numpy as np

F16, Q8, Q4, Q2, Q2K = 0, 1, 2, 3, 4
QBITS = {F16: 16, Q8: 8, Q4: 4, Q2: 2, Q2K: 2}
EPG = {F16: 32, Q8: 64, Q4: 128, Q2: 256, Q2K: 256}
TILE = 16


def _align(n):
    return (n + 255) // 256 * 256


def bpg(enc):
    return EPG[enc] // 32


def scale_record_bytes(enc):
    if enc == Q2K:
        return 20
    return 0 if enc == F16 else 2 * bpg(enc) * (2 if enc == Q2 else 1)


def sections(enc, hidden, ffn):
    """[(code offset, scale offset or None)] per matrix, and the total size."""
    off, out = 0, []
    for n, k in ((ffn, hidden), (ffn, hidden), (hidden, ffn)):
        q = off
        off = _align(off + n * k * QBITS[enc] // 8)
        s = None
        if enc != F16:
            s = off
            off = _align(off + n * (k // EPG[enc]) * scale_record_bytes(enc))
        out.append((q, s))
    if enc == Q2K:                    # padded to the canonical blob's size
        canon = sum(_align(n * k // 4) + _align(n * k // 16) + 2 * _align(n * k // 128)
                    for n, k in ((ffn, hidden), (ffn, hidden), (hidden, ffn)))
        off = max(off, canon)
    return out, off


def within_group(enc, k):
    k = np.asarray(k, dtype=np.int64)
    e = k % EPG[enc]
    t, q, j = (e % 32) // 8, e % 8, e // 32
    if enc == F16:
        return 2 * e, np.zeros_like(k)
    if enc == Q8:
        return 16 * t + 8 * j + q, np.zeros_like(k)
    if enc == Q4:
        return 16 * t + 4 * j + q // 2, 4 * (q % 2)
    return 16 * t + 4 * (j // 2) + 2 * (q // 4) + (j % 2), 2 * (q % 4)


def code_offset(enc, n, k, K):
    n = np.asarray(n, dtype=np.int64)
    k = np.asarray(k, dtype=np.int64)
    G = K // EPG[enc]
    o, shift = within_group(enc, k)
    return 1024 * (G * (n // TILE) + k // EPG[enc]) + 64 * (n % TILE) + o, shift


def scale_offset(enc, n, blk, K, which="d"):
    n = np.asarray(n, dtype=np.int64)
    blk = np.asarray(blk, dtype=np.int64)
    G, b, sb = K // EPG[enc], bpg(enc), scale_record_bytes(enc)
    rec = 16 * sb * (G * (n // TILE) + blk // b) + sb * (n % TILE)
    return rec + 2 * (blk % b) + (2 * b if which == "m" else 0)


def device_matrix(enc, codes_or_f16, d16, m16, n, k):
    """(code section bytes, scale section bytes or None) of one matrix."""
    N, K = np.arange(n)[:, None], np.arange(k)[None, :]
    pos, shift = code_offset(enc, N, K, k)
    if enc == F16:
        bits = np.ascontiguousarray(codes_or_f16, dtype=np.float16).view(np.uint16)
        out = np.zeros(n * k * 2, dtype=np.uint8)
        out[pos.ravel()] = (bits & 0xFF).astype(np.uint8).ravel()
        out[(pos + 1).ravel()] = (bits >> 8).astype(np.uint8).ravel()
        return out, None
    out = np.zeros(n * k * QBITS[enc] // 8, dtype=np.uint8)
    mask = (1 << QBITS[enc]) - 1
    codes = codes_or_f16
    for s in np.unique(shift):
        sel = shift[0] == s
        out[pos[:, sel].ravel()] |= ((codes[:, sel] & mask) << s).astype(np.uint8).ravel()
    sc = np.zeros(n * (k // EPG[enc]) * scale_record_bytes(enc), dtype=np.uint8)
    if enc == Q2K:                    # d16 = (sc bytes [n][k/16], d [n][k/256], dmin [n][k/256])
        scb, dd, dm = d16
        G = k // 256
        grp = np.arange(G)[None, :]
        rec = 16 * 20 * (G * (N // TILE) + grp) + 20 * (N % TILE)
        for arr, o in ((dd, 0), (dm, 2)):
            bits = np.ascontiguousarray(arr, dtype=np.float16).view(np.uint16)
            sc[(rec + o).ravel()] = (bits & 0xFF).astype(np.uint8).ravel()
            sc[(rec + o + 1).ravel()] = (bits >> 8).astype(np.uint8).ravel()
        for j in range(16):
            sc[(rec + 4 + j).ravel()] = scb[:, j::16].ravel()
        return out, sc
    Bk = np.arange(k // 32)[None, :]
    for arr, which in ((d16, "d"), (m16, "m")):
        if arr is None:
            continue
        p = scale_offset(enc, N, Bk, k, which)
        bits = np.ascontiguousarray(arr, dtype=np.float16).view(np.uint16)
        sc[p.ravel()] = (bits & 0xFF).astype(np.uint8).ravel()
        sc[(p + 1).ravel()] = (bits >> 8).astype(np.uint8).ravel()
    return out, sc


def canonical_fields(enc, blob, hidden, ffn):
    """Read a canonical blob back into per-matrix
    (codes or fp16 values, d, m) -- plain row-major unpacking."""
    out, off = [], 0
    for n, k in ((ffn, hidden), (ffn, hidden), (hidden, ffn)):
        if enc == F16:
            w = blob[off:off + n * k * 2].view(np.float16).reshape(n, k)
            off = _align(off + n * k * 2)
            out.append((w, None, None))
            continue
        b = QBITS[enc]
        rows = blob[off:off + n * k * b // 8].reshape(n, k * b // 8)
        off = _align(off + n * k * b // 8)
        kk = np.arange(k)
        codes = (rows[:, kk * b // 8].astype(np.int64) >> ((kk * b) % 8)) & ((1 << b) - 1)
        if enc == Q2K:                # sc [n][k/16] bytes, d and dmin [n][k/256] fp16
            scb = blob[off:off + n * k // 16].reshape(n, k // 16)
            off = _align(off + n * k // 16)
            dd = blob[off:off + n * k // 128].view(np.float16).reshape(n, k // 256)
            off = _align(off + n * k // 128)
            dm = blob[off:off + n * k // 128].view(np.float16).reshape(n, k // 256)
            off = _align(off + n * k // 128)
            out.append((codes, (scb, dd, dm), None))
            continue
        d = blob[off:off + n * k // 16].view(np.float16).reshape(n, k // 32)
        off = _align(off + n * k // 16)
        m = None
        if enc == Q2:
            m = blob[off:off + n * k // 16].view(np.float16).reshape(n, k // 32)
            off = _align(off + n * k // 16)
        out.append((codes, d, m))
    return out


def device_blob(enc, canonical, hidden, ffn):
    """The device-layout blob the library must produce from a canonical one."""
    secs, total = sections(enc, hidden, ffn)
    blob = np.zeros(total, dtype=np.uint8)
    shapes = ((ffn, hidden), (ffn, hidden), (hidden, ffn))
    for (q, s), (n, k), (c, d, m) in zip(secs, shapes,
                                         canonical_fields(enc, canonical, hidden, ffn)):
        code, sc = device_matrix(enc, c, d, m, n, k)
        blob[q:q + code.size] = code
        if sc is not None:
            blob[s:s + sc.size] = sc
    return blob
