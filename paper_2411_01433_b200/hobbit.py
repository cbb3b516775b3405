"""Python API over libhobbit (thin: marshalling of torch tensors / numpy arrays).

    ctx = Context(cfg)                       # hb_create
    ctx.set_router(layer, w_fp16)            # hb_set_router
    ctx.register_expert(l, e, enc, blob)     # hb_register_expert
    ctx.token_begin()                        # hb_token_begin (Eq. 3 T += 1)
    ctx.forward(layer, x, y)                 # moe_layer_forward
    ctx.prefetch(layer, x)                   # prefetch_next_layer
    ctx.load(layer, e, enc)                  # expert_cache_load

PyTorch supplies device memory and streams only.  Tensors passed here must be
contiguous; device tensors must live on the context's device.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from ._lib import (HB_ENC_NONE, HB_F16, HB_HIGH, HB_LOW, HB_Q2, HB_Q4, HB_Q8,  # noqa: F401
                   HB_REG_CANONICAL, HB_REG_DEVICE_BORROW, HB_REG_DEVICE_COPY, HB_REG_HOST_COPY,
                   HB_REG_HOST_PINNED, HB_SKIP, HobbitError, blob_bytes, blob_section,
                   canonical_section, default_config, theta)

check = L.check
lib = L.lib


def _ptr(t) -> C.c_void_p:
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(t.ctypes.data)
    raise TypeError(type(t))


def _nbytes(t) -> int:
    return t.numel() * t.element_size() if isinstance(t, torch.Tensor) else t.nbytes


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Context:
    """One hb_ctx: the expert layer of one model on one GPU (one EP rank)."""

    def __init__(self, cfg: L.hb_config, device: int = 0):
        self.cfg = cfg
        self.device = device
        h = C.c_void_p()
        check(lib.hb_create(C.byref(cfg), device, C.byref(h)))
        self._h = h
        self._keep = []            # host / device buffers that must outlive ctx

    def close(self):
        if self._h is not None and self._h.value:
            lib.hb_destroy(self._h)
        self._h = None
        self._keep = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        return check(rc, self._h)

    # -------------------------------------------------------------- setup
    def set_router(self, layer: int, w):
        on_dev = isinstance(w, torch.Tensor) and w.is_cuda
        if isinstance(w, np.ndarray):
            w = np.ascontiguousarray(w, dtype=np.float16)
        self._check(lib.hb_set_router(self._h, layer, _ptr(w), 1 if on_dev else 0))

    def register_expert(self, layer: int, expert: int, enc: int, blob, flags: int | None = None,
                        canonical: bool = False):
        """Device-layout blobs are borrowed (device / pinned host) or copied;
        canonical=True (SURVEY 8(b) layout, e.g. the oracle's) is always copied
        and converted by the library."""
        if flags is None:
            dev = isinstance(blob, torch.Tensor) and blob.is_cuda
            if canonical:
                flags = HB_REG_DEVICE_COPY if dev else HB_REG_HOST_COPY
            elif dev:
                flags = HB_REG_DEVICE_BORROW
            elif isinstance(blob, torch.Tensor) and blob.is_pinned():
                flags = HB_REG_HOST_PINNED
            else:
                flags = HB_REG_HOST_COPY
            if canonical:
                flags |= HB_REG_CANONICAL
        self._check(lib.hb_register_expert(self._h, layer, expert, enc, _ptr(blob),
                                           _nbytes(blob), flags))
        if (flags & ~HB_REG_CANONICAL) in (HB_REG_DEVICE_BORROW, HB_REG_HOST_PINNED):
            self._keep.append(blob)

    def token_begin(self):
        self._check(lib.hb_token_begin(self._h))

    def reset_sequence(self):
        self._check(lib.hb_reset_sequence(self._h))

    # -------------------------------------------------------------- path
    def forward(self, layer: int, x: torch.Tensor, y: torch.Tensor, stream=None):
        """y[B,H] fp32 <- this rank's Eq. 1 output for x[B,H] fp16 (device)."""
        assert x.dtype == torch.float16 and y.dtype == torch.float32
        self._check(lib.moe_layer_forward(self._h, layer, _ptr(x), x.shape[0], _ptr(y),
                                          _stream(stream)))

    def prefetch(self, layer: int, x: torch.Tensor, stream=None) -> int:
        return self._check(lib.prefetch_next_layer(self._h, layer, _ptr(x), x.shape[0],
                                                   _stream(stream)))

    def load(self, layer: int, expert: int, enc: int, stream=None):
        self._check(lib.expert_cache_load(self._h, layer, expert, enc, _stream(stream)))

    # -------------------------------------------------------------- inspection
    def decisions(self, batch: int):
        n = batch * self.cfg.top_k
        buf = (L.hb_decision * n)()
        got = self._check(lib.hb_get_decisions(self._h, buf, n))
        return [buf[i] for i in range(got)]

    def logits(self, batch: int):
        """Exact router logits of the last forward as Python ints [batch][E]."""
        n = batch * self.cfg.n_experts
        buf = (C.c_int64 * (2 * n))()
        got = self._check(lib.hb_get_logits(self._h, buf, n))
        out = []
        for i in range(got):
            lo, hi = buf[2 * i] & ((1 << 64) - 1), buf[2 * i + 1]
            out.append((hi << 64) + lo)
        E = self.cfg.n_experts
        return [out[b * E:(b + 1) * E] for b in range(batch)]

    def events(self, cap: int = 1 << 16):
        buf = (L.hb_event * cap)()
        got = self._check(lib.hb_get_events(self._h, buf, cap))
        return [buf[i].as_tuple() for i in range(got)]

    # ---- token-sharded EP, staged (hb_config.token_sharded)
    def ts_buffers(self):
        """Device buffers (meta, rows, ret) sized for one exchange direction."""
        m, r, t = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self._check(lib.hb_ts_buffer_bytes(self._h, C.byref(m), C.byref(r), C.byref(t)))
        dev = torch.device("cuda", self.device)
        return (torch.empty(m.value, dtype=torch.uint8, device=dev),
                torch.empty(r.value // 2, dtype=torch.float16, device=dev),
                torch.empty(t.value // 4, dtype=torch.float32, device=dev))

    def ts_dispatch(self, layer: int, x: torch.Tensor, meta_send, rows_send, stream=None):
        self._check(lib.hb_ts_dispatch(self._h, layer, _ptr(x), x.shape[0], _ptr(meta_send),
                                       _ptr(rows_send), _stream(stream)))

    def ts_compute(self, layer: int, meta_recv, rows_recv, ret_send, stream=None):
        self._check(lib.hb_ts_compute(self._h, layer, _ptr(meta_recv), _ptr(rows_recv),
                                      _ptr(ret_send), _stream(stream)))

    def ts_combine(self, ret_recv, y: torch.Tensor, stream=None):
        self._check(lib.hb_ts_combine(self._h, _ptr(ret_recv), y.shape[0], _ptr(y),
                                      _stream(stream)))

    def copy_stats(self):
        """(foreground, background) bytes copied host -> HBM since creation."""
        out = (C.c_uint64 * 2)()
        self._check(lib.hb_copy_stats(self._h, out))
        return int(out[0]), int(out[1])

    def last_expert_bytes(self) -> int:
        v = C.c_uint64()
        self._check(lib.hb_last_expert_bytes(self._h, C.byref(v)))
        return int(v.value)

    def profile(self, max_calls: int):
        """Record K2a/K2b (or K3a/K3b) CUDA events for the next max_calls forwards (0 = off)."""
        self._check(lib.hb_profile(self._h, max_calls))

    def profile_read(self, cap: int = 1 << 16):
        """[(ms_K2a, ms_K2b)] of the recorded forwards (synchronises)."""
        buf = (C.c_float * (2 * cap))()
        n = self._check(lib.hb_profile_read(self._h, buf, cap))
        return [(buf[2 * i], buf[2 * i + 1]) for i in range(n)]

    def stamps(self, max_forwards: int):
        """Arm in-kernel %globaltimer records for the next max_forwards fused forwards (0 = off)."""
        self._check(lib.hb_stamps(self._h, max_forwards))

    def stamps_read(self, cap: int = 1 << 16):
        """[(start, decided, k2a_done, released, end, wg_landed, logits, jobs, h_last, h_first)]
        ns per recorded forward (hb_stamps_read)."""
        buf = (C.c_uint64 * (15 * cap))()
        n = self._check(lib.hb_stamps_read(self._h, buf, cap))
        return [tuple(buf[15 * i:15 * i + 15]) for i in range(n)]

    def nccl_init(self, group=None, tp: bool = False):
        """EP exchange inside the library (A10): rank 0 makes an NCCL unique id,
        torch.distributed broadcasts it, every rank joins; afterwards forward()
        returns the reduced y.  tp=True: the group is the torch.distributed
        group (TP-within-expert, hb_nccl_init_ranks) instead of cfg.rank/world.
        Single process (no process group): world 1."""
        import torch.distributed as dist
        uid = (C.c_char * 128)()
        dist_on = dist.is_available() and dist.is_initialized()
        if not dist_on or dist.get_rank(group) == 0:
            check(lib.hb_nccl_unique_id(uid))
        if dist_on and dist.get_world_size(group) > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0, group=group)
            C.memmove(uid, obj[0], 128)
        if tp:
            n = dist.get_world_size(group) if dist_on else 1
            r = dist.get_rank(group) if dist_on else 0
            self._check(lib.hb_nccl_init_ranks(self._h, uid, n, r))
        else:
            self._check(lib.hb_nccl_init(self._h, uid))

    def broadcast_x(self, x: torch.Tensor, root: int = 0, stream=None):
        """X1: x [B,H] fp16 (device) replicated from EP rank root, in place."""
        assert x.dtype == torch.float16
        self._check(lib.hb_ep_broadcast_x(self._h, _ptr(x), x.shape[0], root, _stream(stream)))

    def set_batched_min(self, min_batch: int):
        """Batches >= min_batch take the tcgen05 grouped-GEMM path K3 (0 = never)."""
        self._check(lib.hb_set_batched_min(self._h, min_batch))

    def launch_count(self) -> int:
        v = C.c_uint64()
        self._check(lib.hb_launch_count(self._h, C.byref(v)))
        return int(v.value)


class HostCache:
    """The library's Eq. 3 cache state machine on the host (no GPU needed)."""

    def __init__(self, cfg: L.hb_config):
        self.cfg = cfg
        h = C.c_void_p()
        check(lib.hbc_create(C.byref(cfg), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.hbc_destroy(self._h)
            self._h = None

    def _check(self, rc):
        if rc < 0:
            raise HobbitError(rc, lib.hbc_last_error(self._h).decode())
        return rc

    def token_begin(self):
        self._check(lib.hbc_token_begin(self._h))

    def reset_sequence(self):
        self._check(lib.hbc_reset_sequence(self._h))

    def forward(self, layer, experts, prec):
        k = self.cfg.top_k
        ex = (C.c_int32 * k)(*experts)
        pr = (C.c_uint8 * k)(*prec)
        out = (C.c_uint8 * k)()
        self._check(lib.hbc_forward(self._h, layer, ex, pr, out))
        return [None if v == HB_ENC_NONE else v for v in out]

    def prefetch(self, layer, predicted):
        """predicted: list over lookahead layers of (experts, prec)."""
        k = self.cfg.top_k
        n = len(predicted)
        ex = (C.c_int32 * max(1, n * k))(*[e for es, _ in predicted for e in es])
        pr = (C.c_uint8 * max(1, n * k))(*[p for _, ps in predicted for p in ps])
        out = C.c_int()
        self._check(lib.hbc_prefetch(self._h, layer, n, ex, pr, C.byref(out)))
        return out.value

    def load(self, layer, expert, enc):
        self._check(lib.hbc_load(self._h, layer, expert, enc))

    def events(self, cap: int = 1 << 16):
        buf = (L.hb_event * cap)()
        got = self._check(lib.hbc_get_events(self._h, buf, cap))
        return [buf[i].as_tuple() for i in range(got)]


# ------------------------------------------------------- device utilities
def quantize_expert(enc: int, w1: torch.Tensor, w3: torch.Tensor, w2: torch.Tensor,
                    out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device blob (uint8) of an fp16 expert in encoding enc (offline quantiser)."""
    ffn, hidden = w1.shape
    nb = blob_bytes(enc, hidden, ffn)
    if out is None:
        out = torch.zeros(nb, dtype=torch.uint8, device=w1.device)
    assert out.numel() == nb
    check(lib.hb_quantize_expert(enc, hidden, ffn, _ptr(w1), _ptr(w3), _ptr(w2), _ptr(out),
                                 _stream(stream)))
    return out


def repack_canonical(enc: int, hidden: int, ffn: int, src: torch.Tensor,
                     out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device-layout blob from a canonical one (both uint8, device)."""
    nb = blob_bytes(enc, hidden, ffn)
    assert src.numel() == nb and src.is_cuda
    if out is None:
        out = torch.zeros(nb, dtype=torch.uint8, device=src.device)
    check(lib.hb_repack_canonical(enc, hidden, ffn, _ptr(src), _ptr(out), _stream(stream)))
    return out


def synth_fill(dst: torch.Tensor, key: int, scale: float, start: int = 0, stream=None):
    """dst (fp16, device) <- the seeded generator's values (synthgen.fill_f16)."""
    assert dst.dtype == torch.float16 and dst.is_cuda
    check(lib.hb_synth_fill_f16(_ptr(dst), dst.numel(), key & ((1 << 64) - 1),
                                float(scale), start, _stream(stream)))
    return dst
