"""Thin Python binding of libtactic.so (include/tactic.h) -- argument marshalling only.

Every step of the decode path runs inside the library's sm_100a kernels; this module
only converts torch tensors / numpy arrays into pointers and the current CUDA stream.
There is no fallback: if the shared library is missing, importing the binding fails.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TACTIC_LIB") or os.path.join(_HERE, "lib", "libtactic.so")  # TACTIC_LIB: A/B experiments

STATUS = {0: "TACTIC_OK", 1: "TACTIC_ERR_INVALID_ARGUMENT", 2: "TACTIC_ERR_SHAPE", 3: "TACTIC_ERR_OOM",
          4: "TACTIC_ERR_CUDA", 5: "TACTIC_ERR_NOT_FINITE", 6: "TACTIC_ERR_UNSUPPORTED"}
FLAG_VALIDATE = 1
FLAG_KMEANS_SIMT = 2
SHARD_GRID_T = 512
SHARD_GRID_STEP = 0.0625
HEAD_DIM = 128


class TacticError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status


class KvDesc(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("group_size", ctypes.c_int32),
                ("seq_len", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("stride_b", ctypes.c_int64),
                ("stride_h", ctypes.c_int64), ("stride_n", ctypes.c_int64)]


class Params(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("init_indices", ctypes.c_void_p), ("flags", ctypes.c_uint32),
                ("num_ctas", ctypes.c_int32), ("exact_frac", ctypes.c_float), ("p1", ctypes.c_float),
                ("p2", ctypes.c_float), ("window_half_frac", ctypes.c_float), ("unit_offset", ctypes.c_int32)]


class SampleConstants(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("x1", ctypes.c_int32), ("x2", ctypes.c_int32), ("w", ctypes.c_int32),
                ("fallback", ctypes.c_int32), ("slots", ctypes.c_int32)]


SAMPLING_KEYS = ("exact_frac", "p1", "p2", "window_half_frac")


def _params(seed=0, init=None, flags=0, num_ctas=0, sampling=None, unit_offset=0) -> Params:
    """tactic_params_t; sampling: optional dict of the Alg. 1 fractions (0 / absent = default)."""
    sampling = dict(sampling or {})
    bad = set(sampling) - set(SAMPLING_KEYS)
    if bad:
        raise ValueError(f"unknown sampling keys {sorted(bad)}")
    return Params(seed, init, flags, num_ctas, *[float(sampling.get(k, 0.0)) for k in SAMPLING_KEYS],
                  int(unit_offset))


class IndexInfo(ctypes.Structure):
    _fields_ = [("units", ctypes.c_int32), ("batch", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("group_size", ctypes.c_int32), ("seq_len", ctypes.c_int32), ("n_clusters", ctypes.c_int32),
                ("iters_requested", ctypes.c_int32), ("select_cluster_size", ctypes.c_int32),
                ("device_bytes", ctypes.c_int64), ("build_gpu_ms", ctypes.c_float)]


_lib = None
_P = ctypes.c_void_p
_I = ctypes.c_int32
_F = ctypes.c_float

_SIGS = {
    "tactic_build_index": [_P, _P, ctypes.POINTER(KvDesc), _I, _I, ctypes.POINTER(Params), _P, ctypes.POINTER(_P)],
    "tactic_index_import": [_P, _P, ctypes.POINTER(KvDesc), _I, _P, _P, ctypes.POINTER(Params), _P,
                            ctypes.POINTER(_P)],
    "tactic_index_export": [_P, _P, _P, _P, _P, _P],
    "tactic_index_info": [_P, ctypes.POINTER(IndexInfo)],
    "tactic_decode": [_P, _P, _F, _P, _P],
    "tactic_decode_ex": [_P, _P, _F, _P, _P, _P],
    "tactic_decode_host": [_P, _P, _F, _P, _P],
    "tactic_decode_debug": [_P, _P, _F, _P, _P, _P, _P, _P, _P, _P],
    "tactic_decode_profiled": [_P, _P, _F, _P, ctypes.POINTER(_P), _I, _P],
    "tactic_decode_attention_only": [_P, _P, _P, _P],
    "tactic_dense_workspace_size": [ctypes.POINTER(KvDesc), _I, ctypes.POINTER(ctypes.c_size_t)],
    "tactic_dense_decode": [_P, _P, _P, ctypes.POINTER(KvDesc), _P, _P, _P, ctypes.c_size_t, _I, _P],
    "tactic_lse_merge": [_P, _P, _I, _I, _P, _P, _P],
    "tactic_decode_stage1": [_P, _P, _P, _P],
    "tactic_decode_stage1b": [_P, _P, _P, _P],
    "tactic_decode_stage2": [_P, _P, _F, _P, _P, _P, _P, _P],
    "tactic_device_check": [ctypes.POINTER(_I)],
    "tactic_index_debug_timing": [_P, _P, _I],
    "tactic_set_tail_capacity": [_P, _I],
    "tactic_append": [_P, _P, _P, _I, _P],
    "tactic_index_tail": [_P, ctypes.POINTER(_I), ctypes.POINTER(_I)],
    "tactic_assign_tokens": [_P, _P, _I, _P, _P],
    "tactic_exact_logits": [_P, _P, _P, _P],
    "tactic_decode_per_head": [_P, _P, _F, _P, _P],
    "tactic_decode_fixed_budget": [_P, _P, _I, _I, _P, _P, _P],
    "tactic_index_set_options": [_P, ctypes.c_uint32],
    "tactic_sample_constants": [_I, ctypes.POINTER(Params), ctypes.POINTER(SampleConstants)],
    "tactic_index_sample_constants": [_P, ctypes.POINTER(SampleConstants)],
}


def lib():
    """Load libtactic.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2502_12216_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.tactic_index_destroy.argtypes = [_P]
        L.tactic_index_destroy.restype = None
        for name in ("tactic_status_string",):
            getattr(L, name).argtypes = [ctypes.c_int]
            getattr(L, name).restype = ctypes.c_char_p
        L.tactic_last_error.argtypes = []
        L.tactic_last_error.restype = ctypes.c_char_p
        L.tactic_version.argtypes = []
        L.tactic_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise TacticError(st, lib().tactic_last_error().decode())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _kv_desc(K: torch.Tensor, group_size: int) -> KvDesc:
    if K.dim() != 4 or K.shape[-1] != HEAD_DIM:
        raise ValueError("K/V must be [B, Hkv, n, 128]")
    if K.dtype != torch.bfloat16 or not K.is_cuda:
        raise ValueError("K/V must be CUDA bfloat16 tensors")
    if K.stride(-1) != 1:
        raise ValueError("last dimension must be contiguous")
    B, H, n, d = K.shape
    return KvDesc(B, H, group_size, n, d, K.stride(0), K.stride(1), K.stride(2))


def version() -> str:
    return lib().tactic_version().decode()


def device_check() -> int:
    n = _I(0)
    _check(lib().tactic_device_check(ctypes.byref(n)))
    return n.value


def _sc_dict(sc: SampleConstants) -> dict:
    return {"N": sc.N, "x1": sc.x1, "x2": sc.x2, "w": sc.w, "fallback": bool(sc.fallback), "slots": sc.slots}


def sample_constants(n: int, sampling: Optional[dict] = None) -> dict:
    """tactic_sample_constants: the integer Alg. 1 sampling constants the library derives
    for n tokens from the sampling fractions (host-only call into the library)."""
    sc = SampleConstants()
    p = _params(sampling=sampling)
    _check(lib().tactic_sample_constants(int(n), ctypes.byref(p), ctypes.byref(sc)))
    return _sc_dict(sc)


class Index:
    """Owns a tactic_index_t (device memory released on close / garbage collection)."""

    def __init__(self, handle: ctypes.c_void_p, K_shape, group_size: int, n_clusters: int):
        self._h = handle
        self.B, self.Hkv, self.n, _ = K_shape
        self.G = group_size
        self.C = n_clusters
        self.units = self.B * self.Hkv

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("index is closed")
        return self._h

    def close(self):
        if self._h is not None and _lib is not None:
            lib().tactic_index_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sample_constants(self) -> dict:
        sc = SampleConstants()
        _check(lib().tactic_index_sample_constants(self.handle, ctypes.byref(sc)))
        return _sc_dict(sc)

    def info(self) -> dict:
        i = IndexInfo()
        _check(lib().tactic_index_info(self.handle, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in IndexInfo._fields_}

    def debug_timing(self) -> np.ndarray:
        """Debug %globaltimer stamps (ns), flat: kernel-specific slots below 1536, the decode
        timeline at 1536 + 4k (TACTIC_TLOG=1 indexes only; see csrc/internal.h)."""
        buf = np.zeros(max(self.units * 128, 8192), dtype=np.uint64)
        _check(lib().tactic_index_debug_timing(self.handle, buf.ctypes.data, buf.size))
        return buf

    def export(self, stream=None) -> dict:
        cent = np.empty((self.units, self.C, HEAD_DIM), dtype=np.float32)
        assign = np.empty((self.units, self.n), dtype=np.int32)
        inertia = np.empty(self.units, dtype=np.float64)
        iters = np.empty(self.units, dtype=np.int32)
        _check(lib().tactic_index_export(self.handle, cent.ctypes.data, assign.ctypes.data, inertia.ctypes.data,
                                         iters.ctypes.data, _stream(stream)))
        return {"centroids": cent, "assign": assign, "inertia": inertia, "iters_run": iters}


def build_index(K: torch.Tensor, V: torch.Tensor, n_clusters: int, iters: int = 10, *, group_size: int = 4,
                seed: int = 0, init: Optional[np.ndarray] = None, flags: int = 0, num_ctas: int = 0,
                sampling: Optional[dict] = None, unit_offset: int = 0, stream=None) -> Index:
    """tactic_build_index: k-means (tcgen05 assignment) + cluster-contiguous KV layout."""
    kv = _kv_desc(K, group_size)
    if tuple(V.shape) != tuple(K.shape) or V.stride() != K.stride() or V.dtype != K.dtype:
        raise ValueError("V must match K in shape, strides and dtype")
    init_arr = None
    if init is not None:
        init_arr = np.ascontiguousarray(init, dtype=np.int32)
        if init_arr.shape != (kv.batch * kv.num_kv_heads, n_clusters):
            raise ValueError("init must be [units, n_clusters]")
    p = _params(seed, init_arr.ctypes.data if init_arr is not None else None, flags, num_ctas, sampling, unit_offset)
    h = ctypes.c_void_p()
    _check(lib().tactic_build_index(_ptr(K), _ptr(V), ctypes.byref(kv), n_clusters, iters, ctypes.byref(p),
                                    _stream(stream), ctypes.byref(h)))
    return Index(h, tuple(K.shape), group_size, n_clusters)


def import_index(K: torch.Tensor, V: torch.Tensor, centroids: np.ndarray, assign: np.ndarray, *,
                 group_size: int = 4, num_ctas: int = 0, sampling: Optional[dict] = None, stream=None) -> Index:
    """tactic_index_import: index from a given clustering (float32 centroids, int32 assignment)."""
    kv = _kv_desc(K, group_size)
    units = kv.batch * kv.num_kv_heads
    cent = np.ascontiguousarray(centroids, dtype=np.float32)
    asg = np.ascontiguousarray(assign, dtype=np.int32)
    if cent.ndim != 3 or cent.shape[0] != units or cent.shape[2] != HEAD_DIM:
        raise ValueError("centroids must be [units, C, 128]")
    if asg.shape != (units, kv.seq_len):
        raise ValueError("assign must be [units, n]")
    C = cent.shape[1]
    p = _params(0, None, 0, num_ctas, sampling)
    h = ctypes.c_void_p()
    _check(lib().tactic_index_import(_ptr(K), _ptr(V), ctypes.byref(kv), C, cent.ctypes.data, asg.ctypes.data,
                                     ctypes.byref(p), _stream(stream), ctypes.byref(h)))
    return Index(h, tuple(K.shape), group_size, C)


def _q_check(q: torch.Tensor, index: Index):
    if q.dtype != torch.bfloat16 or not q.is_cuda or not q.is_contiguous():
        raise ValueError("q must be a contiguous CUDA bfloat16 tensor")
    if q.numel() != index.units * index.G * HEAD_DIM:
        raise ValueError("q must be [B, Hkv*G, 128] for this index")


def decode(q: torch.Tensor, index: Index, p: float, out: Optional[torch.Tensor] = None,
           lse: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """tactic_decode_ex: one decode step of every unit; returns out [B, Hq, 128] bf16."""
    _q_check(q, index)
    if out is None:
        out = torch.empty_like(q)
    _check(lib().tactic_decode_ex(_ptr(q), index.handle, float(p), _ptr(out), _ptr(lse), _stream(stream)))
    return out


def decode_host(q_host: torch.Tensor, index: Index, p: float, out_host: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
    """tactic_decode_host: q and out in host memory (end-to-end call; synchronises)."""
    if q_host.device.type != "cpu" or q_host.dtype != torch.bfloat16 or not q_host.is_contiguous():
        raise ValueError("q_host must be a contiguous CPU bfloat16 tensor")
    if out_host is None:
        out_host = torch.empty_like(q_host)
    _check(lib().tactic_decode_host(_ptr(q_host), index.handle, float(p), _ptr(out_host), _stream(stream)))
    return out_host


def decode_debug(q: torch.Tensor, index: Index, p: float, stream=None) -> dict:
    """tactic_decode_debug: output plus the selection (order, J, fit, union mask) on the host."""
    _q_check(q, index)
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
    U, G, C = index.units, index.G, index.C
    order = np.empty((U, G, C), dtype=np.int32)
    J = np.empty((U, G), dtype=np.int32)
    fit = np.empty((U, G, 6), dtype=np.float64)
    um = np.empty((U, C), dtype=np.uint8)
    _check(lib().tactic_decode_debug(_ptr(q), index.handle, float(p), _ptr(out), _ptr(lse), order.ctypes.data,
                                     J.ctypes.data, fit.ctypes.data, um.ctypes.data, _stream(stream)))
    return {"out": out, "lse": lse, "order": order, "J": J, "fit": fit, "union_mask": um.astype(bool)}


def decode_profiled(q: torch.Tensor, index: Index, p: float, events, out: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
    """tactic_decode_profiled: records 4 torch.cuda.Event objects at the stage boundaries
    (before S1, after S7, after S8, after S9)."""
    _q_check(q, index)
    if out is None:
        out = torch.empty_like(q)
    for e in events:          # torch creates the cudaEvent lazily on first record
        if not e.cuda_event:
            e.record(stream if stream is not None else torch.cuda.current_stream())
    arr = (_P * 4)(*[ctypes.c_void_p(e.cuda_event) for e in events])
    _check(lib().tactic_decode_profiled(_ptr(q), index.handle, float(p), _ptr(out), arr, 4, _stream(stream)))
    return out


def decode_attention_only(q: torch.Tensor, index: Index, out: torch.Tensor, stream=None) -> torch.Tensor:
    """tactic_decode_attention_only: S8 + S9 over the work lists of the last selection on
    this index (measurement aid; run decode with the same q first)."""
    _q_check(q, index)
    _check(lib().tactic_decode_attention_only(_ptr(q), index.handle, _ptr(out), _stream(stream)))
    return out


_ws_cache = {}


def dense_decode(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, out: Optional[torch.Tensor] = None,
                 lse: Optional[torch.Tensor] = None, num_ctas: int = 0, workspace: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    """tactic_dense_decode: the library's own full-attention split-KV baseline."""
    if q.dtype != torch.bfloat16 or not q.is_cuda or not q.is_contiguous() or q.dim() != 3:
        raise ValueError("q must be a contiguous CUDA bfloat16 tensor [B, Hq, 128]")
    if K.dim() != 4 or q.shape[0] != K.shape[0] or q.shape[2] != HEAD_DIM or q.shape[1] % K.shape[1]:
        raise ValueError("q must be [B, Hkv*G, 128] for K [B, Hkv, n, 128]")
    if tuple(V.shape) != tuple(K.shape) or V.stride() != K.stride() or V.dtype != K.dtype:
        raise ValueError("V must match K in shape, strides and dtype")
    G = q.shape[1] // K.shape[1]
    kv = _kv_desc(K, G)
    sz = ctypes.c_size_t()
    _check(lib().tactic_dense_workspace_size(ctypes.byref(kv), num_ctas, ctypes.byref(sz)))
    if workspace is None:
        # the workspace holds self-resetting arrival counters: one per (device, stream)
        s_ = stream if stream is not None else torch.cuda.current_stream(q.device)
        key = (q.device.index, s_.cuda_stream, sz.value)
        workspace = _ws_cache.get(key)
        if workspace is None:
            workspace = torch.zeros(sz.value, dtype=torch.uint8, device=q.device)
            _ws_cache[key] = workspace
    if out is None:
        out = torch.empty_like(q)
    _check(lib().tactic_dense_decode(_ptr(q), _ptr(K), _ptr(V), ctypes.byref(kv), _ptr(out), _ptr(lse),
                                     _ptr(workspace), workspace.numel(), num_ctas, _stream(stream)))
    return out


def dense_workspace_bytes(K: torch.Tensor, group_size: int, num_ctas: int = 0) -> int:
    kv = _kv_desc(K, group_size)
    sz = ctypes.c_size_t()
    _check(lib().tactic_dense_workspace_size(ctypes.byref(kv), num_ctas, ctypes.byref(sz)))
    return sz.value


def lse_merge(o_parts: torch.Tensor, lse_parts: torch.Tensor, out: Optional[torch.Tensor] = None,
              lse: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """tactic_lse_merge: o_parts [S, R, 128] f32, lse_parts [S, R] f32 -> out [R, 128] bf16."""
    S, R = lse_parts.shape
    if out is None:
        out = torch.empty((R, HEAD_DIM), dtype=torch.bfloat16, device=o_parts.device)
    _check(lib().tactic_lse_merge(_ptr(o_parts), _ptr(lse_parts), S, R, _ptr(out), _ptr(lse), _stream(stream)))
    return out


def decode_stage1(q: torch.Tensor, index: Index, local_max: Optional[torch.Tensor] = None, stream=None):
    if local_max is None:
        local_max = torch.empty((index.units, index.G, 2), dtype=torch.float64, device=q.device)
    _check(lib().tactic_decode_stage1(_ptr(q), index.handle, _ptr(local_max), _stream(stream)))
    return local_max


def decode_stage1b(index: Index, global_max: torch.Tensor, mass: Optional[torch.Tensor] = None, stream=None):
    if mass is None:
        mass = torch.empty((index.units, index.G, 1 + SHARD_GRID_T), dtype=torch.float64,
                           device=global_max.device)
    _check(lib().tactic_decode_stage1b(index.handle, _ptr(global_max), _ptr(mass), _stream(stream)))
    return mass


def decode_stage2(q: torch.Tensor, index: Index, p: float, global_max: torch.Tensor, global_mass: torch.Tensor,
                  o_part: Optional[torch.Tensor] = None, lse_part: Optional[torch.Tensor] = None, stream=None):
    if o_part is None:
        o_part = torch.empty((index.units, index.G, HEAD_DIM), dtype=torch.float32, device=q.device)
    if lse_part is None:
        lse_part = torch.empty((index.units, index.G), dtype=torch.float32, device=q.device)
    _check(lib().tactic_decode_stage2(_ptr(q), index.handle, float(p), _ptr(global_max), _ptr(global_mass),
                                      _ptr(o_part), _ptr(lse_part), _stream(stream)))
    return o_part, lse_part


# ------------------------------------------------------------------ multi-step generation
# SURVEY §8(f) NEXT 1; full attention on newly generated tokens, re-clustering
# every 2048 of them; SPEC assign_token.
def _kv_new_check(x: torch.Tensor, index: Index) -> int:
    if x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("new keys / values must be contiguous CUDA bfloat16 tensors")
    if x.dim() != 3 or x.shape[0] != index.units or x.shape[2] != HEAD_DIM:
        raise ValueError("new keys / values must be [units, t, 128]")
    return int(x.shape[1])


def set_tail_capacity(index: Index, capacity: int):
    """tactic_set_tail_capacity: room for `capacity` recent tokens per unit (tail empty)."""
    _check(lib().tactic_set_tail_capacity(index.handle, int(capacity)))


def append(index: Index, k_new: torch.Tensor, v_new: torch.Tensor, stream=None):
    """tactic_append: t new tokens per unit ([units, t, 128] bf16) into the dense tail."""
    t = _kv_new_check(k_new, index)
    if tuple(v_new.shape) != tuple(k_new.shape):
        raise ValueError("v_new must match k_new")
    _kv_new_check(v_new, index)
    _check(lib().tactic_append(index.handle, _ptr(k_new), _ptr(v_new), t, _stream(stream)))


def tail_info(index: Index) -> tuple:
    """(tail length, tail capacity) per unit."""
    n, c = _I(0), _I(0)
    _check(lib().tactic_index_tail(index.handle, ctypes.byref(n), ctypes.byref(c)))
    return n.value, c.value


def assign_tokens(index: Index, k: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """tactic_assign_tokens: nearest centroid (int32 [units, t]) of t new keys per unit."""
    t = _kv_new_check(k, index)
    if out is None:
        out = torch.empty((index.units, t), dtype=torch.int32, device=k.device)
    _check(lib().tactic_assign_tokens(index.handle, _ptr(k), t, _ptr(out), _stream(stream)))
    return out


class DecodeSession:
    """Multi-step decode over one layer's KV cache: the step's new key/value is appended
    to the dense tail of recently generated tokens, then the Tactic decode runs (selected
    clusters plus the whole tail, so the new token attends itself); when the tail is full
    the whole cache (clustered + tail tokens) is re-clustered (B1-B5) with the same
    average cluster size first -- the host policy of P:112.

        s = DecodeSession(K, V, n_clusters=1024, tail_capacity=2048)
        out = s.step(q, k_new, v_new, p=0.9)   # k_new, v_new: [units, 1, 128]
    """

    def __init__(self, K: torch.Tensor, V: torch.Tensor, n_clusters: int, iters: int = 10, *, group_size: int = 4,
                 tail_capacity: int = 2048, seed: int = 0):
        self.B, self.Hkv = K.shape[0], K.shape[1]
        self.G, self.iters, self.seed = group_size, iters, seed
        self.cluster_size = K.shape[2] / n_clusters
        self.tail_capacity = tail_capacity
        self.K, self.V = K.contiguous(), V.contiguous()   # clustered tokens [B, Hkv, n, 128]
        self.k_tail, self.v_tail = [], []                 # appended tokens, [units, t, 128] each
        self.rebuilds = 0
        self._build(n_clusters)

    def _build(self, C: int):
        self.index = build_index(self.K, self.V, C, self.iters, group_size=self.G, seed=self.seed)
        set_tail_capacity(self.index, self.tail_capacity)
        self.k_tail, self.v_tail = [], []

    @property
    def seq_len(self) -> int:
        return self.K.shape[2] + tail_info(self.index)[0]

    def _recluster(self):
        units = self.B * self.Hkv
        kt = torch.cat(self.k_tail, dim=1).view(self.B, self.Hkv, -1, HEAD_DIM)
        vt = torch.cat(self.v_tail, dim=1).view(self.B, self.Hkv, -1, HEAD_DIM)
        assert kt.shape[0] * kt.shape[1] == units
        self.K = torch.cat([self.K, kt], dim=2).contiguous()
        self.V = torch.cat([self.V, vt], dim=2).contiguous()
        C = max(1, min(self.K.shape[2], int(round(self.K.shape[2] / self.cluster_size)), 4096))
        self.index.close()
        self._build(C)
        self.rebuilds += 1

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, p: float,
             out: Optional[torch.Tensor] = None) -> torch.Tensor:
        t = _kv_new_check(k_new, self.index)
        if tail_info(self.index)[0] + t > self.tail_capacity:
            self._recluster()
        append(self.index, k_new, v_new)
        self.k_tail.append(k_new.clone())
        self.v_tail.append(v_new.clone())
        return decode(q, self.index, p, out=out)


# ------------------------------------------------------------------ Table-1 diagnostics
def exact_logits(q: torch.Tensor, index: Index, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """tactic_exact_logits: q . k / sqrt(d) of every clustered token for every query head,
    float32 [units, G, n] in the index's layout order (measurement tooling, NEXT 3)."""
    _q_check(q, index)
    if out is None:
        out = torch.empty((index.units, index.G, index.n), dtype=torch.float32, device=q.device)
    _check(lib().tactic_exact_logits(_ptr(q), index.handle, _ptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------------ per-head loading ablation
def decode_per_head(q: torch.Tensor, index: Index, p: float, out: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
    """tactic_decode_per_head: every query head attends only its own selected clusters
    (NEXT 2 ablation of the GQA union; SPEC own-set normalisation S:421)."""
    _q_check(q, index)
    if out is None:
        out = torch.empty_like(q)
    _check(lib().tactic_decode_per_head(_ptr(q), index.handle, float(p), _ptr(out), _stream(stream)))
    return out


def decode_fixed_budget(q: torch.Tensor, index: Index, budget: int, per_head: bool = False,
                        out: Optional[torch.Tensor] = None, stream=None):
    """tactic_decode_fixed_budget: the Quest-like baseline -- `budget` tokens per head by
    criticality (cluster granularity).  Returns (out, J [units, G])."""
    _q_check(q, index)
    if out is None:
        out = torch.empty_like(q)
    J = np.empty((index.units, index.G), dtype=np.int32)
    _check(lib().tactic_decode_fixed_budget(_ptr(q), index.handle, int(budget), int(bool(per_head)), _ptr(out),
                                            J.ctypes.data, _stream(stream)))
    return out, J


OPT_WINDOWS_EXACT = 1
OPT_CLUSTER_DECODE = 2  # S1-S9 in one launch of per-unit thread-block clusters (decode_fused.cu)
OPT_DETERMINISTIC = 4  # S9 by the partial merge in piece order (bit-reproducible outputs)


def set_options(index: Index, options: int):
    """tactic_index_set_options: selection variants (OPT_WINDOWS_EXACT: SPEC S:284)."""
    _check(lib().tactic_index_set_options(index.handle, int(options)))
