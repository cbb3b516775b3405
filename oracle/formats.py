"""O1 expert-blob decode and the A8 offline quantiser (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper only says experts exist in "int4 / int2 / int8 versions" next to the
fp16/int8 originals (Sec. 5.1 "Configurations"; "replacing a
float16 expert with an int4 version"), built on Llama.cpp.  The bit
formats are therefore OUR reading (readings R7/R8, SURVEY.md 8(c)
A7/A8); real HOBBIT encodings: parity unpinned.

Encodings (block = 32 consecutive elements along K of one row):
    F16  w = the fp16 value
    Q8   w = d * q          q int8 in [-127, 127]          (8.5 bits/weight)
    Q4   w = d * (q - 8)    q in [0, 15]                   (4.5 bits/weight)
    Q2   w = d * q + m      q in [0, 3]                    (3.0 bits/weight)
d, m fp16, one per block.  Every value is an exact dyadic rational in fp64.

Blob of one expert = W1 [F,H], W3 [F,H], W2 [H,F] in that order, each [N,K]
quantised along K (N, K multiples of 256).  Each matrix = a CODE section and
(quantised encodings) a SCALE section, each starting on a 256-byte boundary
of the blob.

Layout.  Rows come in TILES of 16 rows; along K a
row is cut into GROUPS of EPG elements that occupy 64 bytes (EPG = 32 F16,
64 Q8, 128 Q4, 256 Q2; G = K/EPG groups per row).  A UNIT = (tile, group) =
the 16 rows' 64-byte pieces of that group, stored contiguously (1 KB), units
in (tile, group) order:

    code byte of element (n, k) = 1024*(G*tile + grp) + 64*r + o(k % EPG)
        tile = n // 16, r = n % 16, grp = k // EPG

with the within-group offset o (t = (k%32)//8, q = k%8, j = block in group):
    F16: o = 2*(k%32)                  (the group's 32 fp16 values in order)
    Q8 : byte 16*t + 8*j + q                                (whole byte, int8)
    Q4 : byte 16*t + 4*j + q//2, bits 4*(q%2)..+3
    Q2 : byte 16*t + 4*(j//2) + 2*(q//4) + (j%2), bits 2*(q%4)..+1

Scales: one SB-byte record per (unit, row) -- SB = 2*BPG (d of the BPG blocks
of the group, fp16) and, for Q2, another 2*BPG bytes of m:

    scale record of (n, grp) at 16*SB*(G*tile + grp) + SB*r
        d of block j at +2*j,  m of block j at +2*BPG + 2*j   (Q2)

The formulas ARE the definition; tests/golden/formats_*.txt pin them with
bytes worked out by hand.
"""
from __future__ import annotations

import numpy as np

F16, Q8, Q4, Q2 = 0, 1, 2, 3
ENC_NAMES = {F16: "F16", Q8: "Q8", Q4: "Q4", Q2: "Q2"}
QBITS = {F16: 16, Q8: 8, Q4: 4, Q2: 2}
EPG = {F16: 32, Q8: 64, Q4: 128, Q2: 256}      # elements per 64-byte group
BLOCK = 32
TILE = 16
SECTION_ALIGN = 256


def _align(n: int) -> int:
    return (n + SECTION_ALIGN - 1) // SECTION_ALIGN * SECTION_ALIGN


def bpg(enc: int) -> int:
    """Blocks per group."""
    return EPG[enc] // BLOCK


def scale_record_bytes(enc: int) -> int:
    """SB: bytes of scales per (unit, row)."""
    if enc == F16:
        return 0
    return 2 * bpg(enc) * (2 if enc == Q2 else 1)


def matrix_sections(enc: int, n: int, k: int):
    """[(name, nbytes)] of one [n,k] matrix in encoding enc."""
    if enc == F16:
        return [("w", n * k * 2)]
    return [("q", n * k * QBITS[enc] // 8), ("s", n * (k // EPG[enc]) * scale_record_bytes(enc))]


def expert_matrix_shapes(hidden: int, ffn: int):
    """W1 [F,H], W3 [F,H], W2 [H,F] (rows N, reduction K)."""
    return [(ffn, hidden), (ffn, hidden), (hidden, ffn)]


def blob_layout(enc: int, hidden: int, ffn: int):
    """({mat: {section: (offset, nbytes)}}, total bytes) of one expert blob."""
    off = 0
    lay = {}
    for mat, (n, k) in enumerate(expert_matrix_shapes(hidden, ffn)):
        lay[mat] = {}
        for name, nbytes in matrix_sections(enc, n, k):
            lay[mat][name] = (off, nbytes)
            off = _align(off + nbytes)
    return lay, off


def blob_bytes(enc: int, hidden: int, ffn: int) -> int:
    return blob_layout(enc, hidden, ffn)[1]


# ------------------------------------------------------------ code locations

def within_group(enc: int, k):
    """(byte offset inside the row's 64-byte group piece, bit shift) of element k."""
    k = np.asarray(k, dtype=np.int64)
    e = k % EPG[enc]
    t = (e % 32) // 8
    q = e % 8
    j = e // 32
    if enc == F16:
        return 2 * e, np.zeros_like(k)
    if enc == Q8:
        return 16 * t + 8 * j + q, np.zeros_like(k)
    if enc == Q4:
        return 16 * t + 4 * j + q // 2, 4 * (q % 2)
    if enc == Q2:
        return 16 * t + 4 * (j // 2) + 2 * (q // 4) + (j % 2), 2 * (q % 4)
    raise ValueError(enc)


def code_offset(enc: int, n, k, K: int):
    """(byte offset in the code section, bit shift) of element (n, k)."""
    n = np.asarray(n, dtype=np.int64)
    k = np.asarray(k, dtype=np.int64)
    G = K // EPG[enc]
    tile, r = n // TILE, n % TILE
    grp = k // EPG[enc]
    o, shift = within_group(enc, k)
    return 1024 * (G * tile + grp) + 64 * r + o, shift


def scale_offset(enc: int, n, blk, K: int, which: str = "d"):
    """Byte offset in the scale section of d (or m) of block blk of row n."""
    n = np.asarray(n, dtype=np.int64)
    blk = np.asarray(blk, dtype=np.int64)
    G = K // EPG[enc]
    b = bpg(enc)
    tile, r = n // TILE, n % TILE
    grp, j = blk // b, blk % b
    rec = 16 * scale_record_bytes(enc) * (G * tile + grp) + scale_record_bytes(enc) * r
    return rec + 2 * j + (2 * b if which == "m" else 0)


# ------------------------------------------------------------------- decode

def decode_matrix(enc: int, blob: np.ndarray, sections: dict, n: int, k: int) -> np.ndarray:
    """O1: the exact fp64 matrix [n,k] stored in `blob` (uint8) at `sections`."""
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    N = np.arange(n)[:, None]
    Kx = np.arange(k)[None, :]
    if enc == F16:
        off, nb = sections["w"]
        sec = blob[off:off + nb]
        pos, _ = code_offset(enc, N, Kx, k)
        lo = sec[pos].astype(np.uint16)
        hi = sec[pos + 1].astype(np.uint16)
        return (lo | (hi << 8)).view(np.float16).astype(np.float64)
    qoff, qbytes = sections["q"]
    qsec = blob[qoff:qoff + qbytes]
    pos, shift = code_offset(enc, N, Kx, k)
    raw = (qsec[pos].astype(np.int64) >> shift) & ((1 << QBITS[enc]) - 1)
    soff, sbytes = sections["s"]
    ssec = blob[soff:soff + sbytes]

    def f16_at(p):
        return (ssec[p].astype(np.uint16) | (ssec[p + 1].astype(np.uint16) << 8)).view(
            np.float16).astype(np.float64)

    blk = Kx // BLOCK
    d = f16_at(scale_offset(enc, N, blk, k, "d"))
    if enc == Q8:
        q = np.where(raw >= 128, raw - 256, raw)            # two's complement int8
        return d * q
    if enc == Q4:
        return d * (raw - 8)
    m = f16_at(scale_offset(enc, N, blk, k, "m"))
    return d * raw + m


def decode_blob(enc: int, blob: np.ndarray, hidden: int, ffn: int):
    """(W1, W3, W2) in fp64 from one expert blob."""
    lay, total = blob_layout(enc, hidden, ffn)
    assert blob.size >= total, (blob.size, total)
    return tuple(decode_matrix(enc, blob, lay[m], n, k)
                 for m, (n, k) in enumerate(expert_matrix_shapes(hidden, ffn)))


# ---------------------------------------------------------------- quantiser

def quantize_codes(enc: int, w16: np.ndarray):
    """A8 reading: per-block codes and fp16 scale(s) of an fp16 matrix [n,k].

    All arithmetic in IEEE fp32 in exactly this order (the CUDA quantiser
    performs the same operations, so the bytes agree bit for bit):
      Q8: d = f16(amax / 127);  q = clamp(round_half_away(x / d), -127, 127)
      Q4: m = the element of max |x| (first on ties); d = f16(m / -8);
          q = clamp(floor(x / d + 8.5), 0, 15)
      Q2: d = f16((max - min) / 3); m = f16(min);
          q = clamp(round_half_even((x - m) / d), 0, 3)
    d == 0 gives the zero code (Q8 0, Q4 8, Q2 0).
    Returns (codes int64 [n,k], d fp16 [n,k/32], m fp16 [n,k/32] or None).
    """
    n, k = w16.shape
    x = w16.astype(np.float32).reshape(n, k // BLOCK, BLOCK)
    if enc == Q8:
        amax = np.abs(x).max(axis=2)
        d16 = (amax / np.float32(127.0)).astype(np.float16)
        d = d16.astype(np.float32)[..., None]
        with np.errstate(divide="ignore", invalid="ignore"):
            v = x / d
        q = np.sign(v) * np.floor(np.abs(v) + np.float32(0.5))
        q = np.where(d == 0, 0, np.clip(q, -127, 127))
        return q.astype(np.int64).reshape(n, k), d16, None
    if enc == Q4:
        idx = np.abs(x).argmax(axis=2)                      # first on ties
        mval = np.take_along_axis(x, idx[..., None], axis=2)[..., 0]
        d16 = (mval / np.float32(-8.0)).astype(np.float16)
        d = d16.astype(np.float32)[..., None]
        with np.errstate(divide="ignore", invalid="ignore"):
            v = x / d + np.float32(8.5)
        q = np.where(d == 0, 8, np.clip(np.floor(v), 0, 15))
        return q.astype(np.int64).reshape(n, k), d16, None
    if enc == Q2:
        mn = x.min(axis=2)
        mx = x.max(axis=2)
        d16 = ((mx - mn) / np.float32(3.0)).astype(np.float16)
        m16 = mn.astype(np.float16)
        d = d16.astype(np.float32)[..., None]
        with np.errstate(divide="ignore", invalid="ignore"):
            v = (x - m16.astype(np.float32)[..., None]) / d
        q = np.where(d == 0, 0, np.clip(np.rint(v), 0, 3))
        return q.astype(np.int64).reshape(n, k), d16, m16
    raise ValueError(enc)


def pack_codes(enc: int, codes: np.ndarray) -> np.ndarray:
    """Place codes [n,k] at their code_offset; returns the code section (uint8)."""
    n, k = codes.shape
    out = np.zeros(n * k * QBITS[enc] // 8, dtype=np.uint8)
    pos, shift = code_offset(enc, np.arange(n)[:, None], np.arange(k)[None, :], k)
    mask = (1 << QBITS[enc]) - 1
    for s in np.unique(shift):                       # one shift class at a time:
        sel = shift[0] == s                          # no byte repeats inside it
        out[pos[:, sel].ravel()] |= ((codes[:, sel] & mask) << s).astype(np.uint8).ravel()
    return out


def pack_scales(enc: int, d16: np.ndarray, m16) -> np.ndarray:
    """Scale section (uint8) from d [n, k/32] (and m) fp16."""
    n, nb = d16.shape
    k = nb * BLOCK
    out = np.zeros(n * (k // EPG[enc]) * scale_record_bytes(enc), dtype=np.uint8)
    N = np.arange(n)[:, None]
    Bk = np.arange(nb)[None, :]
    for arr, which in ((d16, "d"), (m16, "m")):
        if arr is None:
            continue
        p = scale_offset(enc, N, Bk, k, which)
        bits = arr.view(np.uint16).astype(np.uint16)
        out[p.ravel()] = (bits & 0xFF).astype(np.uint8).ravel()
        out[(p + 1).ravel()] = (bits >> 8).astype(np.uint8).ravel()
    return out


def pack_f16(w16: np.ndarray) -> np.ndarray:
    """F16 code section: the fp16 values at their code_offset."""
    n, k = w16.shape
    out = np.zeros(n * k * 2, dtype=np.uint8)
    pos, _ = code_offset(F16, np.arange(n)[:, None], np.arange(k)[None, :], k)
    bits = np.ascontiguousarray(w16, dtype=np.float16).view(np.uint16)
    out[pos.ravel()] = (bits & 0xFF).astype(np.uint8).ravel()
    out[(pos + 1).ravel()] = (bits >> 8).astype(np.uint8).ravel()
    return out


def quantize_blob(enc: int, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray) -> np.ndarray:
    """One expert blob (uint8) in encoding enc from its fp16 matrices."""
    ffn, hidden = w1.shape
    lay, total = blob_layout(enc, hidden, ffn)
    blob = np.zeros(total, dtype=np.uint8)
    for mat, w in enumerate((w1, w3, w2)):
        sec = lay[mat]
        if enc == F16:
            off, nb = sec["w"]
            blob[off:off + nb] = pack_f16(w)
            continue
        codes, d16, m16 = quantize_codes(enc, w)
        off, nb = sec["q"]
        blob[off:off + nb] = pack_codes(enc, codes)
        off, nb = sec["s"]
        blob[off:off + nb] = pack_scales(enc, d16, m16)
    return blob
