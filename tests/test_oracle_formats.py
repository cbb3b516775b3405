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
    spec = {"bytes": {}, "expect": {}, "mins": None}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "enc":
                spec["enc"] = ENC[tok[1]]
            elif tok[0] == "K":
                spec["K"] = int(tok[1])
            elif tok[0] == "scales":
                spec["scales"] = [int(v, 16) for v in tok[1:]]
            elif tok[0] == "mins":
                spec["mins"] = [int(v, 16) for v in tok[1:]]
            elif tok[0] == "default":
                spec["default"] = int(tok[1], 16)
            elif tok[0] == "byte":
                spec["bytes"][int(tok[1])] = int(tok[2], 16)
            elif tok[0] == "expect":
                spec["expect"][int(tok[1])] = float(tok[2])
    return spec


@pytest.mark.parametrize("name", ["formats_q4.txt", "formats_q2.txt", "formats_q8.txt"])
def test_decode_hand_worked(name):
    # one 16-row tile, one group (K = EPG): row 0's 64 bytes are the first 64
    # bytes of the code section and its scale record the first SB bytes of the
    # scale section (d of each block, then m for Q2); other rows are defaults
    spec = _load_fixture(name)
    enc, K = spec["enc"], spec["K"]
    assert K == fm.EPG[enc]
    q = np.full(16 * 64, spec["default"], dtype=np.uint8)
    for off, v in spec["bytes"].items():
        q[off] = v
    rec = spec["scales"] + (spec["mins"] or [])
    s = np.zeros(16 * fm.scale_record_bytes(enc) // 2, dtype=np.uint16)
    s[:len(rec)] = rec
    blob = np.concatenate([q, s.view(np.uint8)])
    secs = {"q": (0, q.size), "s": (q.size, s.nbytes)}
    w = fm.decode_matrix(enc, blob, secs, 16, K)[0]
    for k, v in spec["expect"].items():
        assert w[k] == v, (name, k, w[k], v)
    if enc == fm.Q4:      # every unlisted element has the default code 8 -> 0
        listed = set(spec["expect"])
        assert all(w[k] == 0.0 for k in range(K) if k not in listed)


def test_fp16_values():
    v = np.array([0x3800, 0x3400, 0xB600, 0x2400, 0x3C00], dtype=np.uint16).view(np.float16)
    assert list(v.astype(np.float64)) == [0.5, 0.25, -0.375, 2.0 ** -6, 1.0]


@pytest.mark.parametrize("enc", [fm.F16, fm.Q8, fm.Q4, fm.Q2])
def test_code_offset_is_a_bijection(enc):
    """Every bit of a 2-tile x 2-group code section is written by exactly one
    element, and every scale byte by exactly one (row, block, d/m)."""
    N, K = 32, 2 * fm.EPG[enc]
    b = fm.QBITS[enc]
    n, k = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    pos, shift = fm.code_offset(enc, n, k, K)
    bits = (pos * 8 + shift)[..., None] + np.arange(b)
    assert np.array_equal(np.sort(bits.ravel()), np.arange(N * K * b))
    if enc == fm.F16:
        return
    nb, blk = np.meshgrid(np.arange(N), np.arange(K // 32), indexing="ij")
    offs = [fm.scale_offset(enc, nb, blk, K, "d")]
    if enc == fm.Q2:
        offs.append(fm.scale_offset(enc, nb, blk, K, "m"))
    allb = np.concatenate([(o[..., None] + np.arange(2)).ravel() for o in offs])
    assert np.array_equal(np.sort(allb), np.arange(N * (K // fm.EPG[enc]) * fm.scale_record_bytes(enc)))


def test_unit_is_contiguous():
    """A unit (16 rows x one group) occupies one contiguous 1 KB of the code section."""
    for enc in (fm.F16, fm.Q8, fm.Q4, fm.Q2):
        K = 4 * fm.EPG[enc]
        n, k = np.meshgrid(np.arange(16, 32), np.arange(2 * fm.EPG[enc], 3 * fm.EPG[enc]),
                           indexing="ij")
        pos, _ = fm.code_offset(enc, n, k, K)
        unit = 1 * 4 + 2                      # tile 1, group 2
        last = pos.max() + (1 if enc == fm.F16 else 0)    # fp16: 2-byte elements
        assert pos.min() == 1024 * unit and last == 1024 * unit + 1023


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
    q = fm.pack_codes(enc, codes)
    s = fm.pack_scales(enc, d16, m16)
    blob = np.concatenate([q, s])
    sec = {"q": (0, q.size), "s": (q.size, s.size)}
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
