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

    Q2K  llama.cpp's Q2_K arithmetic (HOBBIT runs on Llama.cpp,
         whose "int2" version of an int8 model is a k-quant): super-block of
         256 elements of a row = 16 sub-blocks of 16, per sub-block j a byte
         sc_j (low nibble scale, high nibble min), per super-block fp16 d, dmin:
             w = d * (sc_j & 15) * q - dmin * (sc_j >> 4),  q in [0, 3]
         (2.625 bits/weight).  Packed with OUR canonical conventions (LSB-first,
         row-major) rather than llama.cpp's interleaved qs order (R32);
         sections q, sc [n][k/16] bytes, d [n][k/256], dmin [n][k/256].

CANONICAL blob (the interchange format the oracle reads and
writes; the library converts it into its own device layout with
hb_repack_canonical, which the oracle knows nothing about):
one expert = W1 [F,H], W3 [F,H], W2 [H,F] in that order, each [N,K] row-major
and quantised along K.  Per matrix, each section starting on a 256-byte
boundary of the blob:
    F16: "w"  N*K fp16, row-major
    Q*:  "q"  N*K*b/8 bytes, row-major (row stride K*b/8); element k of a row
              sits at bit (k*b) mod 8 of byte floor(k*b/8), LSB first
              (Q4: the low nibble is the even element; Q8: int8 two's complement)
         "d"  N*(K/32) fp16, row-major [N][K/32]
         "m"  N*(K/32) fp16 (Q2 only)
"""
from __future__ import annotations

import numpy as np

F16, Q8, Q4, Q2, Q2K = 0, 1, 2, 3, 4
ENC_NAMES = {F16: "F16", Q8: "Q8", Q4: "Q4", Q2: "Q2", Q2K: "Q2K"}
QBITS = {F16: 16, Q8: 8, Q4: 4, Q2: 2, Q2K: 2}
BLOCK = 32
SUPER, SUB = 256, 16           # Q2K super-block and sub-block
SECTION_ALIGN = 256


def _align(n: int) -> int:
    return (n + SECTION_ALIGN - 1) // SECTION_ALIGN * SECTION_ALIGN


def matrix_sections(enc: int, n: int, k: int):
    """[(name, nbytes)] of one [n,k] matrix in encoding enc."""
    if enc == F16:
        return [("w", n * k * 2)]
    if enc == Q2K:             # codes, sc [n][k/16] bytes, d and dmin [n][k/256] fp16
        return [("q", n * k // 4), ("sc", n * (k // SUB)), ("d", n * (k // SUPER) * 2),
                ("dm", n * (k // SUPER) * 2)]
    secs = [("q", n * k * QBITS[enc] // 8), ("d", n * (k // BLOCK) * 2)]
    if enc == Q2:
        secs.append(("m", n * (k // BLOCK) * 2))
    return secs


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


# ------------------------------------------------------------------- decode

def _f16_section(blob: np.ndarray, sec, n: int, cols: int) -> np.ndarray:
    off, nb = sec
    return blob[off:off + nb].view(np.float16).reshape(n, cols).astype(np.float64)


def decode_matrix(enc: int, blob: np.ndarray, sections: dict, n: int, k: int) -> np.ndarray:
    """O1: the exact fp64 matrix [n,k] stored in `blob` (uint8) at `sections`."""
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    if enc == F16:
        return _f16_section(blob, sections["w"], n, k)
    b = QBITS[enc]
    off, nb = sections["q"]
    rows = blob[off:off + nb].reshape(n, k * b // 8)
    kk = np.arange(k)
    raw = (rows[:, kk * b // 8].astype(np.int64) >> ((kk * b) % 8)) & ((1 << b) - 1)
    if enc == Q2K:             # w = d * (sc & 15) * q - dmin * (sc >> 4)
        off, nb = sections["sc"]
        sc = np.repeat(blob[off:off + nb].reshape(n, k // SUB).astype(np.int64), SUB, axis=1)
        d = np.repeat(_f16_section(blob, sections["d"], n, k // SUPER), SUPER, axis=1)
        dm = np.repeat(_f16_section(blob, sections["dm"], n, k // SUPER), SUPER, axis=1)
        return d * (sc & 15) * raw - dm * (sc >> 4)
    d = np.repeat(_f16_section(blob, sections["d"], n, k // BLOCK), BLOCK, axis=1)
    if enc == Q8:
        return d * np.where(raw >= 128, raw - 256, raw)       # two's complement int8
    if enc == Q4:
        return d * (raw - 8)
    m = np.repeat(_f16_section(blob, sections["m"], n, k // BLOCK), BLOCK, axis=1)
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


def quantize_q2k(w16: np.ndarray):
    """R33: the Q2K quantiser (ours, not llama.cpp's iterative make_qkx2_quants),
    IEEE fp32 in exactly this order (the CUDA quantiser does the same):
      per sub-block j of 16: mn_j = min(0, min x), mx_j = max x,
        s_j = (mx_j - mn_j) / 3,  mm_j = -mn_j
      per super-block: d = f16(max_j s_j / 15), dmin = f16(max_j mm_j / 15)
      sc_lo_j = clamp(rint(s_j / d), 0, 15)   (0 if d == 0)
      sc_hi_j = clamp(rint(mm_j / dmin), 0, 15)  (0 if dmin == 0)
      dl_j = d * sc_lo_j, ml_j = dmin * sc_hi_j
      q = clamp(rint((x + ml_j) / dl_j), 0, 3)  (0 if dl_j == 0)
    Returns (codes int64 [n,k], sc uint8 [n,k/16], d fp16 [n,k/256], dmin fp16 [n,k/256])."""
    n, k = w16.shape
    x = w16.astype(np.float32).reshape(n, k // SUPER, SUPER // SUB, SUB)
    mn = np.minimum(np.float32(0.0), x.min(axis=3))
    mx = x.max(axis=3)
    s_j = (mx - mn) / np.float32(3.0)
    mm_j = -mn
    d16 = (s_j.max(axis=2) / np.float32(15.0)).astype(np.float16)
    dm16 = (mm_j.max(axis=2) / np.float32(15.0)).astype(np.float16)
    d = d16.astype(np.float32)[..., None]
    dm = dm16.astype(np.float32)[..., None]
    with np.errstate(divide="ignore", invalid="ignore"):
        lo = np.where(d == 0, 0, np.clip(np.rint(s_j / d), 0, 15))
        hi = np.where(dm == 0, 0, np.clip(np.rint(mm_j / dm), 0, 15))
        dl = (d * lo.astype(np.float32))[..., None]
        ml = (dm * hi.astype(np.float32))[..., None]
        q = np.where(dl == 0, 0, np.clip(np.rint((x + ml) / dl), 0, 3))
    sc = (lo.astype(np.int64) | (hi.astype(np.int64) << 4)).astype(np.uint8)
    return (q.astype(np.int64).reshape(n, k), sc.reshape(n, k // SUB), d16, dm16)


def pack_codes(enc: int, codes: np.ndarray) -> np.ndarray:
    """The "q" section (uint8): codes [n,k] row-major, LSB first."""
    n, k = codes.shape
    b = QBITS[enc]
    per = 8 // b                                   # codes per byte
    c = (codes.astype(np.int64) & ((1 << b) - 1)).reshape(n, k // per, per)
    out = np.zeros((n, k // per), dtype=np.int64)
    for i in range(per):                           # element per*j + i at bits b*i
        out |= c[:, :, i] << (b * i)
    return out.astype(np.uint8).ravel()


def quantize_blob(enc: int, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray) -> np.ndarray:
    """One canonical expert blob (uint8) in encoding enc from its fp16 matrices."""
    ffn, hidden = w1.shape
    lay, total = blob_layout(enc, hidden, ffn)
    blob = np.zeros(total, dtype=np.uint8)

    def put(sec, arr):
        off, nb = sec
        data = np.ascontiguousarray(arr).view(np.uint8).ravel()
        assert data.size == nb
        blob[off:off + nb] = data

    for mat, w in enumerate((w1, w3, w2)):
        sec = lay[mat]
        if enc == F16:
            put(sec["w"], np.ascontiguousarray(w, dtype=np.float16))
            continue
        if enc == Q2K:
            codes, sc, d16, dm16 = quantize_q2k(w)
            put(sec["q"], pack_codes(enc, codes))
            put(sec["sc"], sc)
            put(sec["d"], d16)
            put(sec["dm"], dm16)
            continue
        codes, d16, m16 = quantize_codes(enc, w)
        put(sec["q"], pack_codes(enc, codes))
        put(sec["d"], d16)
        if enc == Q2:
            put(sec["m"], m16)
    return blob
