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

Blob of one expert = W1 [F,H], W3 [F,H], W2 [H,F] in that order, each row-major
[N,K] quantised along K; each matrix = sections (q, d[, m]); every section
starts on a 256-byte boundary of the blob.  d and m sections are [N, K/32]
fp16 row-major.  The q section is row-major with K*b/8 bytes per row; inside a
row the codes are stored in 64-byte GROUPS, and element k of the row is at

    Q8 : group k//64 , byte 16*t + 8*j + r               (whole byte, int8)
         j = (k%64)//32 , t = (k%32)//8 , r = k%8
    Q4 : group k//128, byte 16*t + 4*j + r//2, bits 4*(r%2)..+3
         j = (k%128)//32, t = (k%32)//8 , r = k%8
    Q2 : group k//256, byte 16*t + 4*(j//2) + 2*(r//4) + (j%2), bits 2*(r%4)..+1
         j = (k%256)//32, t = (k%32)//8 , r = k%8

(byte offsets relative to the group start = row start + 64*group).  The
formulas ARE the definition; tests/golden/formats_*.txt pin them with bytes
worked out by hand.  (Why this order: DESIGN.md "Blob layout".)
"""
from __future__ import annotations

import numpy as np

F16, Q8, Q4, Q2 = 0, 1, 2, 3
ENC_NAMES = {F16: "F16", Q8: "Q8", Q4: "Q4", Q2: "Q2"}
QBITS = {F16: 16, Q8: 8, Q4: 4, Q2: 2}
BLOCK = 32
SECTION_ALIGN = 256


def _align(n: int) -> int:
    return (n + SECTION_ALIGN - 1) // SECTION_ALIGN * SECTION_ALIGN


def matrix_sections(enc: int, n: int, k: int):
    """[(name, nbytes)] of one [n,k] matrix in encoding enc."""
    if enc == F16:
        return [("w", n * k * 2)]
    nb = n * (k // BLOCK) * 2
    q = [("q", n * k * QBITS[enc] // 8), ("d", nb)]
    if enc == Q2:
        q.append(("m", nb))
    return q


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

def code_location(enc: int, k):
    """(byte offset within the row, bit shift) of element k (int or array)."""
    k = np.asarray(k, dtype=np.int64)
    t = (k % 32) // 8
    r = k % 8
    if enc == Q8:
        g, j = k // 64, (k % 64) // 32
        return 64 * g + 16 * t + 8 * j + r, np.zeros_like(k)
    if enc == Q4:
        g, j = k // 128, (k % 128) // 32
        return 64 * g + 16 * t + 4 * j + r // 2, 4 * (r % 2)
    if enc == Q2:
        g, j = k // 256, (k % 256) // 32
        return 64 * g + 16 * t + 4 * (j // 2) + 2 * (r // 4) + (j % 2), 2 * (r % 4)
    raise ValueError(f"no packed codes for encoding {enc}")


def row_group(enc: int) -> int:
    """K must be a multiple of this for encoding enc."""
    return {F16: 32, Q8: 64, Q4: 128, Q2: 256}[enc]


# ------------------------------------------------------------------- decode

def _f16(buf: np.ndarray, off: int, count: int) -> np.ndarray:
    return buf[off:off + 2 * count].view(np.float16)


def decode_matrix(enc: int, blob: np.ndarray, sections: dict, n: int, k: int) -> np.ndarray:
    """O1: the exact fp64 matrix [n,k] stored in `blob` (uint8) at `sections`."""
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    if enc == F16:
        off, _ = sections["w"]
        return _f16(blob, off, n * k).astype(np.float64).reshape(n, k)
    qoff, qbytes = sections["q"]
    rows = blob[qoff:qoff + qbytes].reshape(n, -1)
    byte, shift = code_location(enc, np.arange(k))
    raw = (rows[:, byte].astype(np.int64) >> shift[None, :]) & ((1 << QBITS[enc]) - 1)
    doff, _ = sections["d"]
    d = _f16(blob, doff, n * (k // BLOCK)).astype(np.float64).reshape(n, k // BLOCK)
    d_el = np.repeat(d, BLOCK, axis=1)
    if enc == Q8:
        q = np.where(raw >= 128, raw - 256, raw)            # two's complement int8
        return d_el * q
    if enc == Q4:
        return d_el * (raw - 8)
    moff, _ = sections["m"]
    m = _f16(blob, moff, n * (k // BLOCK)).astype(np.float64).reshape(n, k // BLOCK)
    return d_el * raw + np.repeat(m, BLOCK, axis=1)


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
    """Place codes [n,k] at their code_location; returns uint8 [n, k*b/8]."""
    n, k = codes.shape
    out = np.zeros((n, k * QBITS[enc] // 8), dtype=np.uint8)
    byte, shift = code_location(enc, np.arange(k))
    mask = (1 << QBITS[enc]) - 1
    for s in np.unique(shift):                       # one shift class at a time:
        sel = np.nonzero(shift == s)[0]              # no byte repeats inside it
        out[:, byte[sel]] |= ((codes[:, sel] & mask) << s).astype(np.uint8)
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
            blob[off:off + nb] = np.ascontiguousarray(w, dtype=np.float16).view(np.uint8).ravel()
            continue
        codes, d16, m16 = quantize_codes(enc, w)
        off, nb = sec["q"]
        blob[off:off + nb] = pack_codes(enc, codes).ravel()
        off, nb = sec["d"]
        blob[off:off + nb] = d16.view(np.uint8).ravel()
        if m16 is not None:
            off, nb = sec["m"]
            blob[off:off + nb] = m16.view(np.uint8).ravel()
    return blob
