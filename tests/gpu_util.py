"""Shared helpers for the GPU parity tests (test infrastructure).

Both sides start from the same seeded generator (synthgen/): the CUDA side
draws the fp16 weights with the library's synth kernel and quantises them
with the library's quantiser; the oracle side draws them with numpy and
quantises them with oracle/formats.py.  Nothing the oracle sees comes from
the CUDA path.
"""
from __future__ import annotations

import numpy as np

import synthgen as sg
from oracle import formats as fm
from oracle import moe as om

TOL = 2e-3          # north_star: max relative error (normwise, R12)


def gpu_expert_f16(shape, layer, expert, device="cuda"):
    import torch
    from paper_2411_01433_b200.hobbit import synth_fill
    H, F = shape.hidden, shape.ffn
    out = []
    for mat, (n, k) in enumerate(((F, H), (F, H), (H, F))):
        t = torch.empty(n * k, dtype=torch.float16, device=device)
        key = sg.expert_key(sg.DEFAULT_SEED, layer, expert, mat)
        synth_fill(t, key, float(sg.scale_f32(sg.expert_sigma(shape, mat))))
        out.append(t.view(n, k))
    return out


def gpu_blobs(shape, layer, experts, encs, device="cuda"):
    """{(e, enc): device uint8 blob} built by the library (synth + quantiser)."""
    from paper_2411_01433_b200.hobbit import quantize_expert
    out = {}
    for e in experts:
        w1, w3, w2 = gpu_expert_f16(shape, layer, e, device)
        for enc in encs:
            out[(e, enc)] = quantize_expert(enc, w1, w3, w2)
        del w1, w3, w2
    return out


class OracleStore(om.ExpertStore):
    """Oracle experts: numpy generator + oracle quantiser + oracle decode."""

    def __init__(self, shape):
        self.shape = shape
        self._blobs = {}
        super().__init__(self._blob, shape.hidden, shape.ffn)

    def _blob(self, layer, e, enc):
        key = (layer, e, enc)
        if key not in self._blobs:
            w1, w3, w2 = sg.expert_weights(self.shape, layer, e)
            self._blobs[key] = fm.quantize_blob(enc, w1, w3, w2)
        return self._blobs[key]


def rel_err(y, ref):
    """(normwise max-relative error, elementwise max rel over |ref| >= 0.1 rms)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nw = np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-300)
    rms = np.sqrt((ref ** 2).mean()) if ref.size else 0.0
    sel = (np.abs(ref) >= 0.1 * rms) & (np.abs(ref) > 0)      # an all-zero row has no relative error
    el = (np.abs(y - ref)[sel] / np.abs(ref)[sel]).max() if sel.any() else 0.0
    return nw, el
