"""Thin ctypes binding of libvi.so (include/vi.h): argument marshalling only.

Every step of the memory-step path runs in the library's sm_100a kernels; this module
only converts Python / torch arguments to pointers and status codes to exceptions.
There is no CPU fallback: if libvi.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvi.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2403_16161_b200.build` "
                      "(the memory-step path has no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

VI_OK, VI_NOT_RESIDENT = 0, 1
VI_E_ARG, VI_E_SHAPE, VI_E_CONFIG, VI_E_PROTOCOL, VI_E_CUDA, VI_E_OOM, VI_E_NCCL = -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "VI_OK", 1: "VI_NOT_RESIDENT", -1: "VI_E_ARG", -2: "VI_E_SHAPE", -3: "VI_E_CONFIG",
                -4: "VI_E_PROTOCOL", -5: "VI_E_CUDA", -6: "VI_E_OOM", -7: "VI_E_NCCL"}
DTYPE_BF16, DTYPE_FP32 = 0, 1
FFN_MLP, FFN_F3N = 0, 1
DBG = dict(tokens=0, h=1, q=2, o=3, u=4, g=5, k=6, v=7)

EXPORTS = ["vi_config_default", "vi_create", "vi_create_ex", "vi_destroy", "vi_set_weights", "vi_memory_push",
           "vi_memory_evict", "vi_soft_split", "vi_memory_step", "vi_soft_composite", "vi_refine_commit",
           "vi_memory_state", "vi_run_step", "vi_sync", "vi_last_error", "vi_kernel_launches", "vi_num_slots",
           "vi_stream", "vi_debug_read", "vi_ring_create", "vi_ring_destroy", "vi_ring_push", "vi_ring_evict",
           "vi_ring_commit", "vi_ring_mark_stepped", "vi_ring_state", "vi_version", "vi_memory_step_attn",
           "vi_memory_step_ffn", "vi_tp_layout", "vi_tp_unique_id", "vi_tp_local_allgather", "vi_memory_footprint",
           "vi_memory_read", "vi_ring_create_ex", "vi_run_step_async", "vi_ring_create_refined", "vi_ring_watermark",
           "vi_refined_watermark"]


class ViConfig(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "layers", "heads", "d_model", "tokens_per_frame", "mem_frames", "max_new_frames",
        "feat_h", "feat_w", "feat_c", "kh", "kw", "sh", "sw", "ph", "pw",
        "ffn_hidden", "ffn_kind", "dtype", "pos_embed", "device")] + [("stream", C.c_void_p)] + [
        ("tp_size", C.c_int), ("tp_rank", C.c_int), ("nccl_id", C.c_void_p), ("stream_priority", C.c_int),
        ("ref_rate", C.c_int), ("max_ref_frames", C.c_int), ("win_h", C.c_int), ("win_w", C.c_int),
        ("refined_mem", C.c_int), ("refined_span", C.c_int), ("refined_rate", C.c_int), ("max_refined_refs", C.c_int)]


WEIGHT_FIELDS = ("embed_w", "embed_b", "pos", "ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo", "ln2_g", "ln2_b",
                 "w1", "b1", "w2", "b2", "back_w", "back_b")


class ViWeights(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_float)) for n in WEIGHT_FIELDS]


_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_sig = {
    "vi_config_default": (C.c_int32, [C.POINTER(ViConfig)]),
    "vi_create": (C.c_int32, [C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "vi_create_ex": (C.c_int32, [C.POINTER(_P), C.POINTER(ViConfig)]),
    "vi_destroy": (C.c_int32, [_P]),
    "vi_set_weights": (C.c_int32, [_P, C.POINTER(ViWeights)]),
    "vi_memory_push": (C.c_int32, [_P, C.c_int, _I64P, _I64P, C.POINTER(C.c_int)]),
    "vi_memory_evict": (C.c_int32, [_P, C.c_int64]),
    "vi_soft_split": (C.c_int32, [_P, _P, C.c_int, _P, C.c_int]),
    "vi_memory_step": (C.c_int32, [_P, C.c_int, _P, _P]),
    "vi_soft_composite": (C.c_int32, [_P, _P, C.c_int, _P, C.c_int]),
    "vi_refine_commit": (C.c_int32, [_P, C.c_int64, _P, _P]),
    "vi_memory_state": (C.c_int32, [_P, _I64P, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)]),
    "vi_run_step": (C.c_int32, [_P, _P, C.c_int, _P, _I64P]),
    "vi_run_step_async": (C.c_int32, [_P, _P, C.c_int, _P, _I64P]),
    "vi_sync": (C.c_int32, [_P]),
    "vi_last_error": (C.c_char_p, [_P]),
    "vi_kernel_launches": (C.c_int64, [_P]),
    "vi_num_slots": (C.c_int, [_P]),
    "vi_stream": (_P, [_P]),
    "vi_debug_read": (C.c_int32, [_P, C.c_int, C.c_int, C.c_int, _P, C.c_size_t]),
    "vi_ring_create": (C.c_int32, [C.POINTER(_P), C.c_int, C.c_int]),
    "vi_ring_create_ex": (C.c_int32, [C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int]),
    "vi_ring_create_refined": (C.c_int32, [C.POINTER(_P)] + [C.c_int] * 7),
    "vi_ring_watermark": (C.c_int64, [_P]),
    "vi_refined_watermark": (C.c_int64, [_P]),
    "vi_ring_destroy": (C.c_int32, [_P]),
    "vi_ring_push": (C.c_int32, [_P, C.c_int, _I64P, _I64P, C.POINTER(C.c_int)]),
    "vi_ring_evict": (C.c_int32, [_P, C.c_int64]),
    "vi_ring_commit": (C.c_int32, [_P, C.c_int64]),
    "vi_ring_mark_stepped": (C.c_int32, [_P]),
    "vi_ring_state": (C.c_int32, [_P, _I64P, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)]),
    "vi_version": (C.c_char_p, []),
    "vi_memory_step_attn": (C.c_int32, [_P, C.c_int, _P]),
    "vi_memory_step_ffn": (C.c_int32, [_P, C.c_int, _P, _P]),
    "vi_tp_layout": (C.c_int32, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 5 + [_I64P]),
    "vi_tp_unique_id": (C.c_int32, [_P]),
    "vi_tp_local_allgather": (C.c_int32, [C.POINTER(_P), C.c_int]),
    "vi_memory_footprint": (C.c_int32, [_P, _I64P, _I64P]),
    "vi_memory_read": (C.c_int32, [_P, C.c_int64, _P, _P]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class ViError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    return _lib


def version() -> str:
    return _lib.vi_version().decode()


def _ptr(x) -> Optional[int]:
    """Device or host address of a torch tensor / numpy array (None passes NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous()
        return x.data_ptr()
    return int(x)


# ------------------------------------------------------------------ ring (CUDA-free)
class Ring:
    """vi_ring_*: the integer ring bookkeeping every context uses, without a GPU."""

    def __init__(self, mem_frames: int, max_new_frames: int, ref_rate: int = 0, max_refs: int = 0,
                 refined_span: Optional[int] = None, refined_rate: int = 0, max_refined_refs: int = 0):
        """refined_span = None: no refined memory; s' >= 0: Eq. 4's refined memory."""
        h = _P()
        if refined_span is None:
            st = _lib.vi_ring_create_ex(C.byref(h), mem_frames, max_new_frames, ref_rate, max_refs)
        else:
            st = _lib.vi_ring_create_refined(C.byref(h), mem_frames, max_new_frames, ref_rate, max_refs,
                                             refined_span, refined_rate, max_refined_refs)
        if st != VI_OK:
            raise ViError(st, "vi_ring_create")
        self._h = h
        self.S = mem_frames + max_new_frames + (max_refs if ref_rate > 0 and max_refs > 0 else 0)
        if refined_span is not None:
            self.S += refined_span + 1 + (max_refined_refs if refined_rate > 0 else 0)

    @property
    def watermark(self) -> int:
        return _lib.vi_ring_watermark(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.vi_ring_destroy(self._h)
            self._h = None

    def push(self, n: int) -> Tuple[int, list]:
        first = C.c_int64()
        ev = (C.c_int64 * self.S)()
        nev = C.c_int()
        st = _lib.vi_ring_push(self._h, n, C.byref(first), ev, C.byref(nev))
        if st != VI_OK:
            raise ViError(st, "vi_ring_push")
        return first.value, [ev[i] for i in range(nev.value)]

    def evict(self, fid: int) -> int:
        return _lib.vi_ring_evict(self._h, fid)

    def commit(self, fid: int) -> int:
        return _lib.vi_ring_commit(self._h, fid)

    def mark_stepped(self):
        _lib.vi_ring_mark_stepped(self._h)

    def state(self):
        sid = (C.c_int64 * self.S)()
        ref = (C.c_uint8 * self.S)()
        mask = C.c_uint64()
        _lib.vi_ring_state(self._h, sid, ref, C.byref(mask))
        return list(sid), list(ref), mask.value


# ------------------------------------------------------------------ head sharding
def tp_layout(heads: int, head_dim: int, rows_max: int, tp_size: int, tp_rank: int) -> dict:
    """vi_tp_layout: which heads / query rows rank `tp_rank` of `tp_size` owns and where its
    chunk sits in the head-major gathered buffer (CUDA-free)."""
    v = [C.c_int() for _ in range(5)]
    chunk = C.c_int64()
    st = _lib.vi_tp_layout(heads, head_dim, rows_max, tp_size, tp_rank, *[C.byref(x) for x in v], C.byref(chunk))
    if st != VI_OK:
        raise ViError(st, f"vi_tp_layout(H={heads}, G={tp_size}, r={tp_rank})")
    head0, nheads, qparts, row0, part_rows = (x.value for x in v)
    return dict(head0=head0, nheads=nheads, qparts=qparts, row0=row0, part_rows=part_rows,
                head_rows=qparts * part_rows, chunk_elems=chunk.value)


def tp_unique_id() -> bytes:
    """ncclGetUniqueId through libvi (128 bytes, to broadcast to the other ranks)."""
    buf = C.create_string_buffer(128)
    st = _lib.vi_tp_unique_id(buf)
    if st != VI_OK:
        raise ViError(st, "vi_tp_unique_id")
    return buf.raw


def tp_local_allgather(ctxs) -> None:
    """vi_tp_local_allgather over the contexts of one process (ctxs[r] = rank r)."""
    arr = (_P * len(ctxs))(*[c.handle for c in ctxs])
    st = _lib.vi_tp_local_allgather(arr, len(ctxs))
    if st != VI_OK:
        raise ViError(st, f"vi_tp_local_allgather: {ctxs[0].error()}")


# ------------------------------------------------------------------ context
class Context:
    """One live stream on one GPU (a vi_ctx)."""

    def __init__(self, **cfg):
        k = ViConfig()
        _lib.vi_config_default(C.byref(k))
        stream = cfg.pop("stream", None)
        nccl_id = cfg.pop("nccl_id", None)
        for key, val in cfg.items():
            setattr(k, key, int(val))
        if stream is not None:
            k.stream = stream
        if nccl_id is not None:
            self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128)
            k.nccl_id = C.cast(self._nccl_id, C.c_void_p)
        h = _P()
        st = _lib.vi_create_ex(C.byref(h), C.byref(k))
        if st != VI_OK:
            raise ViError(st, "vi_create_ex failed")
        self._h = h
        self.cfg = k
        self.S = _lib.vi_num_slots(h)

    @classmethod
    def from_synth(cls, c, device: int = 0, stream=None, max_new_frames: Optional[int] = None, tp_size: int = 1,
                   tp_rank: int = 0, nccl_id: Optional[bytes] = None, stream_priority: int = 0) -> "Context":
        """Create from a vi_synth.Config (tp_*: head sharding, see vi.h)."""
        return cls(layers=c.layers, heads=c.heads, d_model=c.d_model, tokens_per_frame=c.tokens,
                   mem_frames=c.mem_frames, max_new_frames=max_new_frames or c.t_new, feat_h=c.feat_h,
                   feat_w=c.feat_w, feat_c=c.feat_c, kh=c.kh, kw=c.kw, sh=c.sh, sw=c.sw, ph=c.ph, pw=c.pw,
                   ffn_hidden=c.ffn_hidden, ffn_kind=c.ffn_kind,
                   dtype=DTYPE_BF16 if c.dtype == "bf16" else DTYPE_FP32, pos_embed=c.pos_embed,
                   device=device, stream=stream, tp_size=tp_size, tp_rank=tp_rank, nccl_id=nccl_id,
                   stream_priority=stream_priority, ref_rate=getattr(c, "ref_rate", 0),
                   max_ref_frames=getattr(c, "max_refs", 0), win_h=getattr(c, "win_h", 0),
                   win_w=getattr(c, "win_w", 0), refined_mem=getattr(c, "refined_mem", 0),
                   refined_span=getattr(c, "refined_span", 0), refined_rate=getattr(c, "refined_rate", 0),
                   max_refined_refs=getattr(c, "max_refined_refs", 0))

    def close(self):
        if getattr(self, "_h", None):
            _lib.vi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def error(self) -> str:
        return _lib.vi_last_error(self._h).decode()

    def _check(self, st: int, what: str, allow=(VI_OK,)) -> int:
        if st not in allow:
            raise ViError(st, f"{what}: {self.error()}")
        return st

    def set_weights(self, w: Dict[str, np.ndarray]):
        keep = {}
        s = ViWeights()
        for f in WEIGHT_FIELDS:
            a = w.get(f)
            if a is None:
                continue
            a = np.ascontiguousarray(a, dtype=np.float32)
            keep[f] = a
            setattr(s, f, a.ctypes.data_as(C.POINTER(C.c_float)))
        self._check(_lib.vi_set_weights(self._h, C.byref(s)), "vi_set_weights")

    def push(self, n: int) -> Tuple[int, list]:
        first = C.c_int64()
        ev = (C.c_int64 * self.S)()
        nev = C.c_int()
        self._check(_lib.vi_memory_push(self._h, n, C.byref(first), ev, C.byref(nev)), "vi_memory_push")
        return first.value, [ev[i] for i in range(nev.value)]

    def evict(self, fid: int) -> int:
        return self._check(_lib.vi_memory_evict(self._h, fid), "vi_memory_evict",
                           allow=(VI_OK, VI_NOT_RESIDENT, VI_E_PROTOCOL, VI_E_ARG))

    def read_kv(self, fid: int, k, v) -> int:
        """vi_memory_read: this context's K/V of a resident past frame into k, v [L][P][Dl]."""
        return self._check(_lib.vi_memory_read(self._h, fid, _ptr(k), _ptr(v)), "vi_memory_read",
                           allow=(VI_OK, VI_NOT_RESIDENT, VI_E_PROTOCOL))

    def commit(self, fid: int, k, v) -> int:
        return self._check(_lib.vi_refine_commit(self._h, fid, _ptr(k), _ptr(v)), "vi_refine_commit",
                           allow=(VI_OK, VI_NOT_RESIDENT, VI_E_PROTOCOL, VI_E_ARG))

    def soft_split(self, feat, n: int, out, project: int):
        self._check(_lib.vi_soft_split(self._h, _ptr(feat), n, _ptr(out), project), "vi_soft_split")

    def memory_step(self, layer: int, x_in, x_out):
        self._check(_lib.vi_memory_step(self._h, layer, _ptr(x_in), _ptr(x_out)), "vi_memory_step")

    def memory_step_attn(self, layer: int, x_in):
        self._check(_lib.vi_memory_step_attn(self._h, layer, _ptr(x_in)), "vi_memory_step_attn")

    def memory_step_ffn(self, layer: int, x_in, x_out):
        self._check(_lib.vi_memory_step_ffn(self._h, layer, _ptr(x_in), _ptr(x_out)), "vi_memory_step_ffn")

    def soft_composite(self, x, n: int, feat, project: int):
        self._check(_lib.vi_soft_composite(self._h, _ptr(x), n, _ptr(feat), project), "vi_soft_composite")

    def run_step_async(self, feat, n: int, out) -> int:
        """vi_run_step_async: enqueue only; host buffers valid / unread until sync()."""
        first = C.c_int64()
        self._check(_lib.vi_run_step_async(self._h, _ptr(feat), n, _ptr(out), C.byref(first)), "vi_run_step_async")
        return first.value

    def run_step(self, feat, n: int, out) -> int:
        first = C.c_int64()
        self._check(_lib.vi_run_step(self._h, _ptr(feat), n, _ptr(out), C.byref(first)), "vi_run_step")
        return first.value

    def state(self):
        sid = (C.c_int64 * self.S)()
        ref = (C.c_uint8 * self.S)()
        mask = C.c_uint64()
        self._check(_lib.vi_memory_state(self._h, sid, ref, C.byref(mask)), "vi_memory_state")
        return list(sid), list(ref), mask.value

    def sync(self):
        self._check(_lib.vi_sync(self._h), "vi_sync")

    def launches(self) -> int:
        return int(_lib.vi_kernel_launches(self._h))

    def footprint(self) -> Tuple[int, int]:
        """(K/V memory bytes, all device bytes owned by the context)."""
        slab, total = C.c_int64(), C.c_int64()
        self._check(_lib.vi_memory_footprint(self._h, C.byref(slab), C.byref(total)), "vi_memory_footprint")
        return slab.value, total.value

    def stream(self) -> int:
        return _lib.vi_stream(self._h)

    def refined_watermark(self) -> int:
        """Eq. 4's watermark t (vi_refined_watermark; -1: no refined frame yet)."""
        return _lib.vi_refined_watermark(self._h)

    def debug_read(self, what: str, dst, layer: int = 0, slot: int = 0):
        nbytes = dst.numel() * dst.element_size() if hasattr(dst, "numel") else dst.nbytes
        self._check(_lib.vi_debug_read(self._h, DBG[what], layer, slot, _ptr(dst), nbytes), "vi_debug_read")
        return dst


PROF_NAMES = ("attention", "gemm", "patch", "row")
_lib.vi_profile.restype = C.c_int32
_lib.vi_profile.argtypes = [_P, C.c_int]
_lib.vi_profile_read.restype = C.c_int32
_lib.vi_profile_read.argtypes = [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
EXPORTS += ["vi_profile", "vi_profile_read"]


def _profile(self, mode: int):
    self._check(_lib.vi_profile(self._h, mode), "vi_profile")


def _profile_read(self):
    ms = (C.c_double * 4)()
    cnt = (C.c_int64 * 4)()
    self._check(_lib.vi_profile_read(self._h, ms, cnt), "vi_profile_read")
    return {n: (ms[i], cnt[i]) for i, n in enumerate(PROF_NAMES)}


Context.profile = _profile
Context.profile_read = _profile_read
