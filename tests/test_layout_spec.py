"""Pins for tests/layout_spec.py, the specification of the library's device
blob layout that the GPU tests hold hb_repack_canonical
to.  Hand-worked bytes at a unit with tile >= 1, row != 0 and group >= 1, a
bijection check and unit contiguity."""
import numpy as np
import pytest

from tests import layout_spec as ls


@pytest.mark.parametrize("enc", [ls.F16, ls.Q8, ls.Q4, ls.Q2])
def test_code_offset_is_a_bijection(enc):
    """Every bit of a 2-tile x 2-group code section is written by exactly one
    element, and every scale byte by exactly one (row, block, d/m)."""
    N, K = 32, 2 * ls.EPG[enc]
    b = ls.QBITS[enc]
    n, k = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    pos, shift = ls.code_offset(enc, n, k, K)
    bits = (pos * 8 + shift)[..., None] + np.arange(b)
    assert np.array_equal(np.sort(bits.ravel()), np.arange(N * K * b))
    if enc == ls.F16:
        return
    nb, blk = np.meshgrid(np.arange(N), np.arange(K // 32), indexing="ij")
    offs = [ls.scale_offset(enc, nb, blk, K, "d")]
    if enc == ls.Q2:
        offs.append(ls.scale_offset(enc, nb, blk, K, "m"))
    allb = np.concatenate([(o[..., None] + np.arange(2)).ravel() for o in offs])
    assert np.array_equal(np.sort(allb), np.arange(N * (K // ls.EPG[enc]) * ls.scale_record_bytes(enc)))


def test_unit_is_contiguous():
    """A unit (16 rows x one group) occupies one contiguous 1 KB of the code section."""
    for enc in (ls.F16, ls.Q8, ls.Q4, ls.Q2):
        K = 4 * ls.EPG[enc]
        n, k = np.meshgrid(np.arange(16, 32), np.arange(2 * ls.EPG[enc], 3 * ls.EPG[enc]),
                           indexing="ij")
        pos, _ = ls.code_offset(enc, n, k, K)
        unit = 1 * 4 + 2                      # tile 1, group 2
        last = pos.max() + (1 if enc == ls.F16 else 0)
        assert pos.min() == 1024 * unit and last == 1024 * unit + 1023


# (enc, K, n, k) -> (byte offset, bit shift), worked by hand from the formulas:
#   Q4, K = 256 (G = 2): n = 21 -> tile 1, r = 5; k = 130 -> grp 1, e = 2:
#     t = 0, q = 2, j = 0 -> o = 1, shift 0; 1024*(2*1 + 1) + 64*5 + 1 = 3393
#   Q4, n = 21, k = 255 -> grp 1, e = 127: t = 3, q = 7, j = 3 ->
#     o = 48 + 12 + 3 = 63, shift 4; 3072 + 320 + 63 = 3455
#   Q2, K = 512 (G = 2): n = 17 -> tile 1, r = 1; k = 300 -> grp 1, e = 44:
#     j = 1, t = 1, q = 4 -> o = 16 + 0 + 2 + 1 = 19, shift 0; 3072 + 64 + 19 = 3155
#   Q8, K = 128 (G = 2): n = 30 -> tile 1, r = 14; k = 100 -> grp 1, e = 36:
#     j = 1, t = 0, q = 4 -> o = 8 + 4 = 12; 3072 + 896 + 12 = 3980
#   F16, K = 64 (G = 2): n = 16 -> tile 1, r = 0; k = 33 -> grp 1, o = 2 -> 3072 + 2
HAND = [(ls.Q4, 256, 21, 130, 3393, 0), (ls.Q4, 256, 21, 255, 3455, 4),
        (ls.Q2, 512, 17, 300, 3155, 0), (ls.Q8, 128, 30, 100, 3980, 0),
        (ls.F16, 64, 16, 33, 3074, 0)]


@pytest.mark.parametrize("enc,K,n,k,off,shift", HAND)
def test_code_offset_hand_worked(enc, K, n, k, off, shift):
    o, s = ls.code_offset(enc, n, k, K)
    assert (int(o), int(s)) == (off, shift)


def test_scale_offset_hand_worked():
    """Q2, K = 512 (G = 2, BPG = 8, SB = 32): row 17 (tile 1, r = 1), block 13
    (grp 1, j = 5): record 16*32*(2 + 1) + 32*1 = 1568; d at +10 = 1578,
    m at +16 + 10 = 1594.  Q4, K = 256 (SB = 8): row 21 (tile 1, r 5), block 6
    (grp 1, j 2): 16*8*3 + 8*5 + 4 = 428."""
    assert int(ls.scale_offset(ls.Q2, 17, 13, 512, "d")) == 1578
    assert int(ls.scale_offset(ls.Q2, 17, 13, 512, "m")) == 1594
    assert int(ls.scale_offset(ls.Q4, 21, 6, 256, "d")) == 428


def test_device_blob_size_equals_canonical():
    from oracle import formats as fm
    for enc in (ls.F16, ls.Q8, ls.Q4, ls.Q2):
        for H, F in ((256, 512), (4096, 14336), (4096, 6400)):
            assert ls.sections(enc, H, F)[1] == fm.blob_bytes(enc, H, F)
