"""Pins for oracle/formats.py (O1 decode, A8 quantiser, blob layout).

Pins are things other than the oracle itself: bytes worked out by hand
(tests/golden/formats_*.txt), closed-form sizes against the paper's Table 1,
and invariants of the quantiser (round-trip error bound).
"""
import os

import numpy as np
import pytest

from oracle import formats as fm
from tests.conftest import GOLDEN

ENC = {"F16": fm.F16, "Q8": fm.Q8, "Q4": fm.Q4, "Q2": fm.Q2}


def _load_fixture(name):
    spec = {"bytes": {}, "expect": {}, "d": {}, "m": {}}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "enc":
                spec["enc"] = ENC[tok[1]]
            elif tok[0] in ("N", "K"):
                spec[tok[0]] = int(tok[1])
            elif tok[0] in ("d", "m"):
                spec[tok[0]][(int(tok[1]), int(tok[2]))] = int(tok[3], 16)
            elif tok[0] == "default":
                spec["default"] = int(tok[1], 16)
            elif tok[0] == "byte":
                spec["bytes"][int(tok[1])] = int(tok[2], 16)
            elif tok[0] == "expect":
                spec["expect"][(int(tok[1]), int(tok[2]))] = float(tok[3])
    return spec


@pytest.mark.parametrize("name", ["formats_q4.txt", "formats_q2.txt", "formats_q8.txt"])
def test_decode_hand_worked(name):
    """Canonical sections built from the fixture (code bytes, d/m per (row,
    block)) decode to the hand-worked values, rows 0 and 1, blocks 0 and 1."""
    spec = _load_fixture(name)
    enc, N, K = spec["enc"], spec["N"], spec["K"]
    q = np.full(N * K * fm.QBITS[enc] // 8, spec["default"], dtype=np.uint8)
    for off, v in spec["bytes"].items():
        q[off] = v
    secs, parts, off = {"q": (0, q.size)}, [q], q.size
    for which in ("d", "m"):
        if not spec[which]:
            continue
        a = np.zeros((N, K // 32), dtype=np.uint16)
        for (r, b), v in spec[which].items():
            a[r, b] = v
        secs[which] = (off, a.nbytes)
        parts.append(a.view(np.uint8).ravel())
        off += a.nbytes
    w = fm.decode_matrix(enc, np.concatenate(parts), secs, N, K)
    for (r, k), v in spec["expect"].items():
        assert w[r, k] == v, (name, r, k, w[r, k], v)
    if enc == fm.Q4:      # every unlisted element has the default code 8 -> 0
        listed = set(spec["expect"])
        assert all(w[r, k] == 0.0 for r in range(N) for k in range(K) if (r, k) not in listed)


def test_fp16_values():
    v = np.array([0x3800, 0x3400, 0xB600, 0x2400, 0x3C00], dtype=np.uint16).view(np.float16)
    assert list(v.astype(np.float64)) == [0.5, 0.25, -0.375, 2.0 ** -6, 1.0]


def test_pack_codes_lsb_first_worked_example():
    """element k at bit (k*b) mod 8 of byte floor(k*b/8).
    Q4 codes (1, 2, 3, 4) -> bytes 0x21, 0x43; Q2 codes (1, 2, 3, 0, 3, ...) ->
    0b00_11_10_01 = 0x39 then 0x03; Q8 -5 -> 0xFB (two's complement)."""
    assert list(fm.pack_codes(fm.Q4, np.array([[1, 2, 3, 4] + [8] * 28]))[:2]) == [0x21, 0x43]
    assert list(fm.pack_codes(fm.Q2, np.array([[1, 2, 3, 0, 3] + [0] * 27]))[:2]) == [0x39, 0x03]
    assert fm.pack_codes(fm.Q8, np.array([[-5] + [0] * 31]))[0] == 0xFB


def test_f16_section_worked_example():
    """F16 canonical section: element (1, 3) of a [2, 32] matrix is the fp16
    at byte offset 2*(32*1 + 3) = 70, little endian; 0x3C00 -> 1.0."""
    sec = np.zeros(2 * 32 * 2, dtype=np.uint8)
    sec[70], sec[71] = 0x00, 0x3C
    w = fm.decode_matrix(fm.F16, sec, {"w": (0, sec.size)}, 2, 32)
    assert w[1, 3] == 1.0 and np.count_nonzero(w) == 1


def test_quantiser_q4_worked_example():
    """block with max-magnitude -1.0 -> d = 0.125; 0.5 -> 12,
    0.25 -> 10, 0 -> 8, -1.0 -> 0, each dequantising to itself."""
    x = np.zeros((1, 32), dtype=np.float16)
    x[0, :4] = [0.5, 0.25, 0.0, -1.0]
    codes, d, _ = fm.quantize_codes(fm.Q4, x)
    assert float(d[0, 0]) == 0.125
    assert list(codes[0, :4]) == [12, 10, 8, 0]
    blob = fm.quantize_blob(fm.Q4, np.zeros((256, 128), np.float16),
                            np.zeros((256, 128), np.float16), np.zeros((128, 256), np.float16))
    assert blob.size == fm.blob_bytes(fm.Q4, 128, 256)


def test_quantiser_q8_ties_round_half_away():
    """A8 reading (Q8 round-half-away, as ggml's roundf).  Block with amax
    127/128 -> d = f16(127/128 / 127) = 2^-7 exactly; x/d is exact in fp32:
    x = 2.5 d -> 3 (half-even would give 2), -2.5 d -> -3, 0.5 d -> 1 (half-even 0),
    -0.5 d -> -1, 3.5 d -> 4, 1.25 d -> 1, amax -> 127."""
    d = 2.0 ** -7
    vals = [127 * d, 2.5 * d, -2.5 * d, 0.5 * d, -0.5 * d, 3.5 * d, 1.25 * d]
    x = np.zeros((1, 32), dtype=np.float16)
    x[0, :len(vals)] = vals
    assert all(float(a) == b for a, b in zip(x[0, :len(vals)], vals))   # fp16-exact inputs
    codes, d16, _ = fm.quantize_codes(fm.Q8, x)
    assert float(d16[0, 0]) == d
    assert list(codes[0, :len(vals)]) == [127, 3, -3, 1, -1, 4, 1]


def test_quantiser_q2_ties_round_half_even():
    """A8 reading (Q2 round-half-even).  Block min 0, max 3 -> d = f16(3/3) = 1,
    m = 0; (x - m)/d = x: 0.5 -> 0 (half-away would give 1), 1.5 -> 2,
    2.5 -> 2 (half-away 3), 2.75 -> 3, 3 -> 3."""
    vals = [0.0, 3.0, 0.5, 1.5, 2.5, 2.75, 0.25]
    x = np.zeros((1, 32), dtype=np.float16)
    x[0, :len(vals)] = vals
    codes, d16, m16 = fm.quantize_codes(fm.Q2, x)
    assert float(d16[0, 0]) == 1.0 and float(m16[0, 0]) == 0.0
    assert list(codes[0, :len(vals)]) == [0, 3, 0, 2, 2, 3, 0]


def test_quantiser_q4_ties_floor_plus_half():
    """A8 reading (Q4 q = floor(x/d + 8.5), ggml Q4_0).  Block max-magnitude
    -1.0 -> d = -1/-8 = 0.125: x/d = 0.5 (x = 0.0625) -> floor(9.0) = 9;
    x/d = -0.5 (x = -0.0625) -> floor(8.0) = 8; x/d = 1.5 -> 10; x/d = -1.5 -> 7;
    +1.0 -> x/d = 8 -> floor(16.5) = 16 -> clamp 15."""
    vals = [-1.0, 0.0625, -0.0625, 0.1875, -0.1875, 1.0]
    x = np.zeros((1, 32), dtype=np.float16)
    x[0, :len(vals)] = vals
    codes, d16, _ = fm.quantize_codes(fm.Q4, x)
    assert float(d16[0, 0]) == 0.125
    assert list(codes[0, :len(vals)]) == [0, 9, 8, 10, 7, 15]


def test_quantiser_zero_block_codes():
    z = np.zeros((1, 64), np.float16)
    for enc, zero in ((fm.Q8, 0), (fm.Q4, 8), (fm.Q2, 0)):
        codes, d, _ = fm.quantize_codes(enc, z)
        assert np.all(codes == zero) and np.all(d.astype(np.float32) == 0)


@pytest.mark.parametrize("enc", [fm.Q8, fm.Q4, fm.Q2])
def test_quantiser_roundtrip_bound(enc):
    """|x - deq(q(x))| <= d/2 (+ the fp16 rounding of d) on random blocks."""
    rng = np.random.default_rng(7)
    n, k = 64, 512
    w = (rng.standard_normal((n, k)) * 0.02).astype(np.float16)
    codes, d16, m16 = fm.quantize_codes(enc, w)
    parts = [fm.pack_codes(enc, codes), d16.view(np.uint8).ravel()]
    if m16 is not None:
        parts.append(m16.view(np.uint8).ravel())
    blob = np.concatenate(parts)
    sizes = [p.size for p in parts]
    sec = {"q": (0, sizes[0]), "d": (sizes[0], sizes[1])}
    if m16 is not None:
        sec["m"] = (sizes[0] + sizes[1], sizes[2])
    deq = fm.decode_matrix(enc, blob, sec, n, k)
    # and the decode reproduces the codes' own dequantisation element-wise
    dd = np.repeat(d16.astype(np.float64), 32, axis=1)
    own = {fm.Q8: dd * codes, fm.Q4: dd * (codes - 8),
           fm.Q2: dd * codes + (np.repeat(m16.astype(np.float64), 32, axis=1) if m16 is not None else 0)}[enc]
    assert np.array_equal(deq, own)
    d = np.abs(np.repeat(d16.astype(np.float64), 32, axis=1))
    err = np.abs(deq - w.astype(np.float64))
    # scale rounding: d carries a relative error <= 2^-11, which can move the
    # largest code's reconstruction by up to qmax * d * 2^-11
    qmax = {fm.Q8: 127, fm.Q4: 8, fm.Q2: 3}[enc]
    bound = d * (0.5 + qmax * 2.0 ** -10) + 1e-12
    if enc == fm.Q4:
        # Q4_0 is asymmetric: the code range is [-8, 7], so x/d near +8
        # clips to 7 and may be off by up to one step d
        clipped = codes == 15
        assert np.all(err[clipped] <= d[clipped] * (1 + qmax * 2.0 ** -10) + 1e-12)
        assert np.all(err[~clipped] <= bound[~clipped])
    else:
        assert np.all(err <= bound)


def test_blob_sizes_match_paper_table1():
    """Table 1 (tab:moe-model): expert weights 84 GB / 75 GB; with
    H=4096, F=14336 (Mixtral) / 6400 (Phi) in fp16 these are exactly 84 and 75 GiB."""
    mix = 32 * 8 * fm.blob_bytes(fm.F16, 4096, 14336)
    phi = 32 * 16 * fm.blob_bytes(fm.F16, 4096, 6400)
    assert mix == 84 * 2 ** 30
    assert phi == 75 * 2 ** 30


def test_blob_sizes_closed_form():
    """SURVEY 8(a) A5 byte counts: sections are 256-aligned with no padding."""
    assert fm.blob_bytes(fm.F16, 4096, 14336) == 352_321_536
    assert fm.blob_bytes(fm.Q8, 4096, 14336) == 187_170_816
    assert fm.blob_bytes(fm.Q4, 4096, 14336) == 99_090_432
    assert fm.blob_bytes(fm.Q2, 4096, 14336) == 66_060_288
    assert fm.blob_bytes(fm.F16, 4096, 6400) == 157_286_400
    assert fm.blob_bytes(fm.Q4, 4096, 6400) == 44_236_800
    assert fm.blob_bytes(fm.Q2, 4096, 6400) == 29_491_200
    # bits per weight: 16, 8.5, 4.5, 3.0
    n = 3 * 4096 * 14336
    assert [fm.blob_bytes(e, 4096, 14336) * 8 / n for e in (0, 1, 2, 3)] == [16, 8.5, 4.5, 3.0]


def test_f16_blob_roundtrip():
    rng = np.random.default_rng(3)
    w1 = rng.standard_normal((64, 32)).astype(np.float16)
    w3 = rng.standard_normal((64, 32)).astype(np.float16)
    w2 = rng.standard_normal((32, 64)).astype(np.float16)
    out = fm.decode_blob(fm.F16, fm.quantize_blob(fm.F16, w1, w3, w2), 32, 64)
    for a, b in zip(out, (w1, w3, w2)):
        assert np.array_equal(a, b.astype(np.float64))


# ---------------------------------------------------------------- Q2K (R32/R33)
def _q2k_blob(codes, sc, d16, dm16):
    """One [1, 256] Q2K matrix laid out by hand: codes LSB first (4 per byte),
    then the 16 sub-block bytes, then d, then dmin."""
    q = np.zeros(64, dtype=np.uint8)
    for k, c in enumerate(codes):
        q[k // 4] |= (c & 3) << (2 * (k % 4))
    parts = [q, np.asarray(sc, dtype=np.uint8), np.array([d16], dtype=np.float16).view(np.uint8),
             np.array([dm16], dtype=np.float16).view(np.uint8)]
    sec, off = {}, 0
    for name, part in zip(("q", "sc", "d", "dm"), parts):
        sec[name] = (off, part.size)
        off += part.size
    return np.concatenate(parts), sec


def test_q2k_decode_hand_worked():
    """Q2K (llama.cpp's Q2_K arithmetic): element k of a super-block lies in
    sub-block j = k // 16; sc_j = j | (15 - j) << 4, q = k % 4, d = 0.5,
    dmin = 0.25.  Values worked out by hand:
      k = 0   (j = 0, q = 0):  0.5*0*0  - 0.25*15 = -3.75
      k = 17  (j = 1, q = 1):  0.5*1*1  - 0.25*14 = -3.0
      k = 130 (j = 8, q = 2):  0.5*8*2  - 0.25*7  =  6.25
      k = 255 (j = 15, q = 3): 0.5*15*3 - 0.25*0  = 22.5"""
    codes = [k % 4 for k in range(256)]
    sc = [j | ((15 - j) << 4) for j in range(16)]
    blob, sec = _q2k_blob(codes, sc, 0.5, 0.25)
    w = fm.decode_matrix(fm.Q2K, blob, sec, 1, 256)
    assert w[0, 0] == -3.75 and w[0, 17] == -3.0 and w[0, 130] == 6.25 and w[0, 255] == 22.5


def test_q2k_quantiser_exact_when_representable():
    """Values on the Q2K grid of d = 0.5, sc_lo = 15 (dl = 7.5), no negative
    part (dmin = 0): every sub-block holds 0, 7.5, 15, 22.5 and round-trips
    exactly (the quantiser picks d = max s_j / 15 = 7.5 / 15 = 0.5)."""
    row = np.array([7.5 * (k % 4) for k in range(512)], dtype=np.float16)[None, :]
    codes, sc, d16, dm16 = fm.quantize_q2k(row)
    assert np.all(d16 == 0.5) and np.all(dm16 == 0) and np.all(sc == 15)
    assert np.array_equal(codes[0], np.arange(512) % 4)


def test_q2k_quantiser_roundtrip_bound_and_container():
    """|x - deq| <= dl_j / 2 + the scale roundings, on random rows; the blob
    size is the closed form of its four sections."""
    rng = np.random.default_rng(11)
    w = (rng.standard_normal((32, 512)) * 0.02).astype(np.float16)
    codes, sc, d16, dm16 = fm.quantize_q2k(w)
    parts = [fm.pack_codes(fm.Q2K, codes), sc.ravel(), d16.view(np.uint8).ravel(),
             dm16.view(np.uint8).ravel()]
    sec, off = {}, 0
    for name, part in zip(("q", "sc", "d", "dm"), parts):
        sec[name] = (off, part.size)
        off += part.size
    deq = fm.decode_matrix(fm.Q2K, np.concatenate(parts), sec, 32, 512)
    dl = np.repeat(np.repeat(d16.astype(np.float64), 16, axis=1) * (sc & 15), 16, axis=1)
    x = w.astype(np.float64)
    ml = np.repeat(np.repeat(dm16.astype(np.float64), 16, axis=1) * (sc >> 4), 16, axis=1)
    inside = (x >= -ml) & (x <= 3 * dl - ml)
    err = np.abs(deq - x)
    # a 4-bit scale step can leave the sub-block range up to 1/30 of the super-block max outside
    slack = np.repeat(np.repeat(np.maximum(d16, dm16).astype(np.float64), 256, axis=1), 1, axis=0)
    assert np.all(err[inside] <= 0.5 * dl[inside] + 1e-12)
    assert np.all(err <= 0.5 * dl + 3 * slack + 1e-12)
    # 2.625 bits per weight: q + sc + d + dmin, each section 256-aligned
    n_k = [(14336, 4096), (14336, 4096), (4096, 14336)]
    assert fm.blob_bytes(fm.Q2K, 4096, 14336) == sum(n * k // 4 + n * k // 16 + 2 * (n * k // 128)
                                                      for n, k in n_k)
