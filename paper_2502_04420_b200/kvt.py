"""Thin Python binding of libkvt.so (include/kvt.h) — argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module only checks torch
tensors (dtype, device, contiguity), passes raw pointers and the current CUDA stream through
ctypes, and raises ``KvtError`` with the library's message on a non-zero status.  There is no CPU
fallback: if ``libkvt.so`` is missing, importing this module fails loudly.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

import torch

import os

# KVT_LIB selects an alternative build (kernel A/B experiments: libkvt_<variant>.so); default libkvt.so
_LIB_PATH = Path(__file__).resolve().parent / os.environ.get("KVT_LIB", "libkvt.so")

MODE_PER_TOKEN_ASYM = 0
MODE_KIVI = 1
MODE_PER_CHANNEL_ASYM = 2      # kvt_layer_sensitivity only (A28)
_MODE_NAMES = {"per-token-asym": MODE_PER_TOKEN_ASYM, "kivi": MODE_KIVI}


class KvtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"kvt status {status}: {msg}")
        self.status = status


class _Spec(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("key_bits", ctypes.c_int32), ("value_bits", ctypes.c_int32),
                ("group", ctypes.c_int32), ("residual", ctypes.c_int32)]


class _Cache(ctypes.Structure):
    _fields_ = [("spec", _Spec), ("batch", ctypes.c_int32), ("kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("capacity", ctypes.c_int32),
                ("k_codes", ctypes.c_void_p), ("k_meta", ctypes.c_void_p), ("k_resid", ctypes.c_void_p),
                ("v_codes", ctypes.c_void_p), ("v_meta", ctypes.c_void_p), ("v_resid", ctypes.c_void_p),
                ("block_table", ctypes.c_void_p), ("max_pages", ctypes.c_int32), ("num_pages", ctypes.c_int32)]


class _Pair(ctypes.Structure):
    _fields_ = [("key_bits", ctypes.c_int32), ("value_bits", ctypes.c_int32)]


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python paper_2502_04420_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(_LIB_PATH))
    P, i32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64
    sig = {
        "kvt_abi_version": (ctypes.c_uint32, []),
        "kvt_status_string": (ctypes.c_char_p, [i32]),
        "kvt_last_error": (ctypes.c_char_p, []),
        "kvt_config_load": (i32, [ctypes.c_char_p, ctypes.POINTER(P)]),
        "kvt_config_num_layers": (i32, [P]),
        "kvt_config_layer": (i32, [P, i32, ctypes.POINTER(_Spec)]),
        "kvt_config_equivalent_bits": (ctypes.c_double, [P]),
        "kvt_config_label_bits": (ctypes.c_double, [P]),
        "kvt_config_model_name": (ctypes.c_char_p, [P]),
        "kvt_config_free": (None, [P]),
        "kvt_validate_spec": (i32, [ctypes.POINTER(_Spec), i32]),
        "kvt_cache_buffer_sizes": (i32, [ctypes.POINTER(_Spec), i32, i32, i32, i32, ctypes.POINTER(u64)]),
        "kvt_quantize_append": (i32, [ctypes.POINTER(_Cache), P, P, ctypes.POINTER(ctypes.c_int64), P, P, P, P,
                                      i32, P]),
        "kvt_decode_workspace_bytes": (i32, [ctypes.POINTER(_Cache), i32, P, ctypes.POINTER(u64)]),
        "kvt_decode_plan": (i32, [ctypes.POINTER(_Cache), i32, P, ctypes.POINTER(i32)]),
        "kvt_decode_attention": (i32, [ctypes.POINTER(_Cache), P, i32, P, P, ctypes.c_float, P, i32, P, u64, P]),
        "kvt_append_decode_attention": (i32, [ctypes.POINTER(_Cache), P, P, ctypes.POINTER(ctypes.c_int64), P, P, i32,
                                              P, i32, P, ctypes.c_float, P, i32, P, u64, P]),
        "kvt_decode_attention_partial": (i32, [ctypes.POINTER(_Cache), P, i32, P, P, ctypes.c_float, P, P, u64,
                                               P]),
        "kvt_decode_attention_partial_push": (i32, [ctypes.POINTER(_Cache), P, i32, P, P, ctypes.c_float,
                                                    ctypes.POINTER(P), i32, P, u64, P]),
        "kvt_combine_partials": (i32, [P, i32, i32, i32, i32, P, i32, P]),
        "kvt_sensitivity_workspace_bytes": (i32, [i32, i32, i32, i32, i32, i32, ctypes.POINTER(u64)]),
        "kvt_layer_sensitivity": (i32, [i32, i32, i32, P, i32, i32, i32, P, P, i32, i32, i32, ctypes.c_float,
                                        ctypes.POINTER(_Pair), i32, P, P, u64, P]),
        "kvt_page_bytes": (i32, [ctypes.POINTER(_Spec), i32, i32, ctypes.POINTER(u64)]),
        "kvt_pareto_prune": (i32, [ctypes.POINTER(_Pair), P, i32, P]),
        "kvt_dbscan": (i32, [P, i32, i32, ctypes.c_double, i32, P]),
        "kvt_prune_and_cluster": (i32, [ctypes.POINTER(_Pair), i32, P, i32, ctypes.c_double, i32, P, P,
                                        ctypes.POINTER(i32)]),
        "kvt_search_space_log10": (i32, [P, i32, ctypes.POINTER(ctypes.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
ABI_VERSION = int(_lib.kvt_abi_version())
EXPORTED = ("kvt_abi_version", "kvt_status_string", "kvt_last_error", "kvt_config_load", "kvt_config_num_layers",
            "kvt_config_layer", "kvt_config_equivalent_bits", "kvt_config_label_bits", "kvt_config_model_name",
            "kvt_config_free", "kvt_validate_spec", "kvt_cache_buffer_sizes", "kvt_quantize_append",
            "kvt_decode_workspace_bytes", "kvt_decode_attention", "kvt_decode_attention_partial",
            "kvt_combine_partials", "kvt_sensitivity_workspace_bytes", "kvt_layer_sensitivity",
            "kvt_pareto_prune", "kvt_dbscan", "kvt_prune_and_cluster", "kvt_search_space_log10", "kvt_page_bytes",
            "kvt_decode_attention_partial_push", "kvt_append_decode_attention", "kvt_decode_plan")


def lib():
    return _lib


def _check(status: int):
    if status != 0:
        raise KvtError(status, _lib.kvt_last_error().decode())


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    return t


def _check_lengths(cache: "LayerCache", t: torch.Tensor, name: str):
    """int32 CUDA tensor with at least `batch` entries (the kernels read batch of them)."""
    _dev(t, name, torch.int32)
    if not t.is_contiguous() or t.numel() < cache.batch:
        raise ValueError(f"{name} must be a contiguous int32 tensor with >= {cache.batch} entries")


def _check_q(cache: "LayerCache", q: torch.Tensor) -> int:
    """q must be [batch][g * kv_heads][head_dim] for this cache; returns H_q."""
    if q.dim() != 3 or q.shape[0] != cache.batch or q.shape[2] != cache.head_dim or q.shape[1] % cache.kv_heads:
        raise ValueError(f"q must be [batch={cache.batch}][g*{cache.kv_heads}][{cache.head_dim}], got {tuple(q.shape)}")
    return q.shape[1]


def _check_new(cache: "LayerCache", k_new: torch.Tensor, v_new: torch.Tensor):
    _dev(k_new, "k_new", torch.bfloat16)
    _dev(v_new, "v_new", torch.bfloat16)
    if k_new.dim() != 4 or k_new.shape[0] != cache.batch or k_new.shape[1] != cache.kv_heads \
            or k_new.shape[3] != cache.head_dim:
        raise ValueError(f"k_new must be [batch={cache.batch}][kv_heads={cache.kv_heads}][T][{cache.head_dim}], "
                         f"got {tuple(k_new.shape)}")
    if k_new.shape != v_new.shape or k_new.stride() != v_new.stride() or k_new.stride(-1) != 1:
        raise ValueError("k_new and v_new need the same shape/strides with a contiguous last dim")


def _check_out(t: torch.Tensor, shape, name: str):
    if not t.is_cuda or not t.is_contiguous() or t.numel() < math.prod(shape):
        raise ValueError(f"{name} must be a contiguous CUDA tensor of {list(shape)} elements")


def _host_i32(t) -> Optional[ctypes.Array]:
    if t is None:
        return None
    vals = [int(v) for v in (t.tolist() if isinstance(t, torch.Tensor) else t)]
    return (ctypes.c_int32 * len(vals))(*vals)


# ------------------------------------------------------------------------------------------------
# a1: configuration
# ------------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class LayerSpec:
    mode: int
    key_bits: int
    value_bits: int
    group: int = 32
    residual: int = 0

    def _c(self) -> _Spec:
        return _Spec(self.mode, self.key_bits, self.value_bits, self.group, self.residual)

    @staticmethod
    def kivi(key_bits, value_bits, group=32, residual=32):
        return LayerSpec(MODE_KIVI, key_bits, value_bits, group, residual)

    @staticmethod
    def per_token(key_bits, value_bits, group=32, residual=0):
        return LayerSpec(MODE_PER_TOKEN_ASYM, key_bits, value_bits, group, residual)


class Config:
    """A searched layer-wise configuration (kvt_config_load)."""

    def __init__(self, path_or_json: str):
        h = ctypes.c_void_p()
        _check(_lib.kvt_config_load(str(path_or_json).encode(), ctypes.byref(h)))
        self._h = h
        self.num_layers = int(_lib.kvt_config_num_layers(h))
        self.equivalent_bits = float(_lib.kvt_config_equivalent_bits(h))
        self.label_bits = float(_lib.kvt_config_label_bits(h))
        self.model_name = _lib.kvt_config_model_name(h).decode()
        self.layers = []
        for i in range(self.num_layers):
            s = _Spec()
            _check(_lib.kvt_config_layer(h, i, ctypes.byref(s)))
            self.layers.append(LayerSpec(s.mode, s.key_bits, s.value_bits, s.group, s.residual))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.kvt_config_free(h)
            self._h = None


def load_config(path_or_json: str) -> Config:
    return Config(path_or_json)


def validate_spec(spec: LayerSpec, head_dim: int = 128):
    s = spec._c()
    _check(_lib.kvt_validate_spec(ctypes.byref(s), head_dim))


def cache_buffer_sizes(spec: LayerSpec, batch: int, kv_heads: int, head_dim: int, capacity: int):
    out = (ctypes.c_uint64 * 6)()
    s = spec._c()
    _check(_lib.kvt_cache_buffer_sizes(ctypes.byref(s), batch, kv_heads, head_dim, capacity, out))
    return [int(v) for v in out]


BUFFER_NAMES = ("k_codes", "k_meta", "k_resid", "v_codes", "v_meta", "v_resid")


def page_bytes(spec: "LayerSpec", kv_heads: int, head_dim: int = 128) -> int:
    """Bytes of one page (kv_heads tile records of 32 tokens) of a paged cache (include/kvt.h)."""
    out = ctypes.c_uint64()
    _check(_lib.kvt_page_bytes(ctypes.byref(spec._c()), kv_heads, head_dim, ctypes.byref(out)))
    return int(out.value)


class LayerCache:
    """One layer's packed cache; the six buffers are torch uint8 tensors owned here.

    Paged (vLLM-style) when `block_table` is given: an int32 [batch][max_pages] device tensor mapping
    32-token block j of sequence b to a page of a pool of `num_pages` pages (k_codes); capacity is then
    32 * max_pages.  The caller owns the table and its allocation policy."""

    def __init__(self, spec: LayerSpec, batch: int, kv_heads: int, head_dim: int, capacity: int,
                 device="cuda", block_table: Optional[torch.Tensor] = None, num_pages: Optional[int] = None):
        self.spec, self.batch, self.kv_heads, self.head_dim, self.capacity = spec, batch, kv_heads, head_dim, capacity
        sizes = cache_buffer_sizes(spec, batch, kv_heads, head_dim, capacity)
        self.block_table = block_table
        if block_table is not None:
            _dev(block_table, "block_table", torch.int32)
            if block_table.dim() != 2 or block_table.shape[0] != batch or not block_table.is_contiguous():
                raise ValueError("block_table must be a contiguous int32 [batch][max_pages] tensor")
            if capacity != 32 * block_table.shape[1]:
                raise ValueError("paged cache: capacity must be 32 * max_pages")
            if not num_pages or num_pages < 1:
                raise ValueError("paged cache: num_pages >= 1 required")
            sizes = list(sizes)
            sizes[0] = num_pages * page_bytes(spec, kv_heads, head_dim)
        self.num_pages = num_pages if block_table is not None else 0
        self.sizes = dict(zip(BUFFER_NAMES, sizes))
        self.buffers = {n: (torch.empty(max(sz, 16), dtype=torch.uint8, device=device) if sz else None)
                        for n, sz in self.sizes.items()}
        self._c = _Cache(spec._c(), batch, kv_heads, head_dim, capacity,
                         *[(b.data_ptr() if b is not None else None) for b in self.buffers.values()],
                         block_table.data_ptr() if block_table is not None else None,
                         block_table.shape[1] if block_table is not None else 0, self.num_pages)

    def slice_view(self, name: str, b: int, h: int) -> torch.Tensor:
        """Bytes of buffer `name` for (batch row b, kv head h)."""
        per = self.sizes[name] // (self.batch * self.kv_heads)
        off = (b * self.kv_heads + h) * per
        return self.buffers[name][off:off + per]

    @property
    def nbytes(self) -> int:
        return sum(self.sizes.values())


# ------------------------------------------------------------------------------------------------
# a2/a3: quantise on append
# ------------------------------------------------------------------------------------------------
def quantize_append(cache: LayerCache, k_new: torch.Tensor, v_new: torch.Tensor, len_before: torch.Tensor,
                    n_new: torch.Tensor, len_before_host=None, n_new_host=None, n_new_max: Optional[int] = None,
                    stream=None):
    """k_new/v_new: bf16 [B][H][T][d] (d contiguous); len_before/n_new: int32 [B] on the device."""
    _check_new(cache, k_new, v_new)
    _check_lengths(cache, len_before, "len_before")
    _check_lengths(cache, n_new, "n_new")
    strides = (ctypes.c_int64 * 3)(k_new.stride(0), k_new.stride(1), k_new.stride(2))
    if n_new_max is None:
        n_new_max = k_new.shape[2]
    _check(_lib.kvt_quantize_append(ctypes.byref(cache._c), _ptr(k_new), _ptr(v_new), strides,
                                    _host_i32(len_before_host), _ptr(len_before), _host_i32(n_new_host),
                                    _ptr(n_new), int(n_new_max), ctypes.c_void_p(_stream(stream))))


# ------------------------------------------------------------------------------------------------
# a4/a5: decode attention
# ------------------------------------------------------------------------------------------------
def decode_plan(cache: LayerCache, n_q_heads: int, seq_len_host=None) -> dict:
    """The work plan decode_attention would use (kvt_decode_plan): kernel, CTAs, whole units per SM of the per-SM
    plan (0: none), resident CTAs per SM."""
    out = (ctypes.c_int32 * 4)()
    _check(_lib.kvt_decode_plan(ctypes.byref(cache._c), n_q_heads, _host_i32(seq_len_host), out))
    return {"kernel": "tensor-core" if out[0] == 1 else "generic", "ctas": int(out[1]), "sm_whole_units": int(out[2]),
            "ctas_per_sm": int(out[3])}


def decode_workspace_bytes(cache: LayerCache, n_q_heads: int, seq_len_host=None) -> int:
    out = ctypes.c_uint64()
    _check(_lib.kvt_decode_workspace_bytes(ctypes.byref(cache._c), n_q_heads, _host_i32(seq_len_host),
                                           ctypes.byref(out)))
    return int(out.value)


def decode_attention(cache: LayerCache, q: torch.Tensor, seq_len: torch.Tensor, seq_len_host=None,
                     scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
                     out_dtype=torch.float32, workspace: Optional[torch.Tensor] = None, stream=None):
    """q: bf16 [B][H_q][d]; seq_len: int32 [B] (device).  Returns out [B][H_q][d] (fp32 or bf16)."""
    _dev(q, "q", torch.bfloat16)
    _check_lengths(cache, seq_len, "seq_len")
    H_q = _check_q(cache, q)
    q = q.contiguous()
    B, _, d = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)                          # A9
    if out is None:
        out = torch.empty(B, H_q, d, dtype=out_dtype, device=q.device)
    od = 1 if out.dtype == torch.float32 else 0
    if out.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("out must be a contiguous fp32 or bf16 tensor")
    _check_out(out, (B, H_q, d), "out")
    if workspace is None:
        nb = decode_workspace_bytes(cache, H_q, seq_len_host)
        workspace = torch.zeros(max(nb, 16), dtype=torch.uint8, device=q.device)   # counters start at zero
    _check(_lib.kvt_decode_attention(ctypes.byref(cache._c), _ptr(q), H_q, _host_i32(seq_len_host), _ptr(seq_len),
                                     float(scale), _ptr(out), od, _ptr(workspace), workspace.numel(),
                                     ctypes.c_void_p(_stream(stream))))
    return out


def append_decode_attention(cache: LayerCache, k_new: torch.Tensor, v_new: torch.Tensor, len_before: torch.Tensor,
                            n_new: torch.Tensor, q: torch.Tensor, seq_len: torch.Tensor, n_new_max: int = 1,
                            scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
                            out_dtype=torch.float32, workspace: Optional[torch.Tensor] = None, stream=None):
    """One layer's serving step (kvt_append_decode_attention): append k_new/v_new [B][H][T][d] (n_new[b] <= T
    tokens of each sequence, T <= n_new_max) and attend with q over seq_len (= len_before + n_new, the caller's)
    tokens.  No host lengths: capturable once in a CUDA graph."""
    _check_new(cache, k_new, v_new)
    for t, n in ((len_before, "len_before"), (n_new, "n_new"), (seq_len, "seq_len")):
        _check_lengths(cache, t, n)
    _dev(q, "q", torch.bfloat16)
    H_q = _check_q(cache, q)
    q = q.contiguous()
    B, _, d = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if out is None:
        out = torch.empty(B, H_q, d, dtype=out_dtype, device=q.device)
    if out.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("out must be a contiguous fp32 or bf16 tensor")
    _check_out(out, (B, H_q, d), "out")
    if workspace is None:
        nb = decode_workspace_bytes(cache, H_q, None)
        workspace = torch.zeros(max(nb, 16), dtype=torch.uint8, device=q.device)
    strides = (ctypes.c_int64 * 3)(k_new.stride(0), k_new.stride(1), k_new.stride(2))
    _check(_lib.kvt_append_decode_attention(ctypes.byref(cache._c), _ptr(k_new), _ptr(v_new), strides, _ptr(len_before),
                                            _ptr(n_new), int(n_new_max), _ptr(q), H_q, _ptr(seq_len), float(scale),
                                            _ptr(out), 1 if out.dtype == torch.float32 else 0, _ptr(workspace),
                                            workspace.numel(), ctypes.c_void_p(_stream(stream))))
    return out


def decode_attention_partial(cache: LayerCache, q: torch.Tensor, seq_len: torch.Tensor, seq_len_host=None,
                             scale: Optional[float] = None, partial: Optional[torch.Tensor] = None,
                             workspace: Optional[torch.Tensor] = None, stream=None):
    """Partial (m, l, o) fp32 [B][H_q][d + 2] over this shard's tokens (a6)."""
    _dev(q, "q", torch.bfloat16)
    _check_lengths(cache, seq_len, "seq_len")
    H_q = _check_q(cache, q)
    q = q.contiguous()
    B, _, d = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if partial is None:
        partial = torch.empty(B, H_q, d + 2, dtype=torch.float32, device=q.device)
    _dev(partial, "partial", torch.float32)
    _check_out(partial, (B, H_q, d + 2), "partial")
    if workspace is None:
        nb = decode_workspace_bytes(cache, H_q, seq_len_host)
        workspace = torch.zeros(max(nb, 16), dtype=torch.uint8, device=q.device)
    _check(_lib.kvt_decode_attention_partial(ctypes.byref(cache._c), _ptr(q), H_q, _host_i32(seq_len_host),
                                             _ptr(seq_len), float(scale), _ptr(partial), _ptr(workspace),
                                             workspace.numel(), ctypes.c_void_p(_stream(stream))))
    return partial


def decode_attention_partial_push(cache: LayerCache, q: torch.Tensor, seq_len: torch.Tensor, dsts,
                                  seq_len_host=None, scale: Optional[float] = None,
                                  workspace: Optional[torch.Tensor] = None, stream=None):
    """a6 with the exchange fused into the kernel: the partial (m, l, o) rows [B][H_q][d + 2] are stored into
    every destination of `dsts` (1..8 fp32 tensors, or raw device addresses, e.g. this shard's slot of each
    peer's symmetric-memory gathered buffer)."""
    _dev(q, "q", torch.bfloat16)
    _check_lengths(cache, seq_len, "seq_len")
    H_q = _check_q(cache, q)
    q = q.contiguous()
    B, _, d = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    ptrs = []
    for t in dsts:
        if isinstance(t, torch.Tensor):
            if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous() or t.numel() < B * H_q * (d + 2):
                raise ValueError("push destinations must be contiguous fp32 CUDA tensors of [B][H_q][d + 2]")
            ptrs.append(t.data_ptr())
        else:
            ptrs.append(int(t))
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    if workspace is None:
        nb = decode_workspace_bytes(cache, H_q, seq_len_host)
        workspace = torch.zeros(max(nb, 16), dtype=torch.uint8, device=q.device)
    _check(_lib.kvt_decode_attention_partial_push(ctypes.byref(cache._c), _ptr(q), H_q, _host_i32(seq_len_host),
                                                  _ptr(seq_len), float(scale), arr, len(ptrs), _ptr(workspace),
                                                  workspace.numel(), ctypes.c_void_p(_stream(stream))))


def combine_partials(gathered: torch.Tensor, out: Optional[torch.Tensor] = None, out_dtype=torch.float32,
                     stream=None):
    """gathered: fp32 [N][B][H_q][d + 2] → out [B][H_q][d]."""
    _dev(gathered, "gathered", torch.float32)
    gathered = gathered.contiguous()
    N, B, H_q, d2 = gathered.shape
    d = d2 - 2
    if out is None:
        out = torch.empty(B, H_q, d, dtype=out_dtype, device=gathered.device)
    od = 1 if out.dtype == torch.float32 else 0
    _check(_lib.kvt_combine_partials(_ptr(gathered), N, B, H_q, d, _ptr(out), od, ctypes.c_void_p(_stream(stream))))
    return out


# ------------------------------------------------------------------------------------------------
# a7: layer sensitivity
# ------------------------------------------------------------------------------------------------
ERROR_NAMES = ("e_k", "e_v", "e_a", "e_o", "e_o_l1")


def layer_sensitivity(mode: int, group: int, residual: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                      q_pos0: int, pairs: Sequence[tuple], scale: Optional[float] = None, stream=None):
    """q bf16 [H_q][T_q][d]; k, v bf16 [H_kv][S][d] → fp64 [n_pairs][5] on the device."""
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _dev(t, n, torch.bfloat16)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    H_q, T_q, d = q.shape
    H_kv, S, _ = k.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    cp = (_Pair * len(pairs))(*[_Pair(int(a), int(b)) for a, b in pairs])
    nb = ctypes.c_uint64()
    _check(_lib.kvt_sensitivity_workspace_bytes(H_q, T_q, H_kv, S, d, group, ctypes.byref(nb)))
    ws = torch.empty(max(int(nb.value), 16), dtype=torch.uint8, device=q.device)
    out = torch.empty(len(pairs), 5, dtype=torch.float64, device=q.device)
    _check(_lib.kvt_layer_sensitivity(mode, group, residual, _ptr(q), H_q, T_q, q_pos0, _ptr(k), _ptr(v), H_kv, S,
                                      d, float(scale), cp, len(pairs), _ptr(out), _ptr(ws), ws.numel(),
                                      ctypes.c_void_p(_stream(stream))))
    return out


# ------------------------------------------------------------------------------------------------
# search-space pruning after calibration (host only): App. D
# ------------------------------------------------------------------------------------------------
def _pairs(pairs: Sequence[tuple]):
    return (_Pair * len(pairs))(*[_Pair(int(a), int(b)) for a, b in pairs])


def _f64(a) -> "np.ndarray":
    import numpy as np
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def pareto_prune(pairs: Sequence[tuple], e_o) -> list:
    """Intra-layer pruning: True for the pairs on the (equivalent bits, e_o) Pareto frontier."""
    import numpy as np
    e = _f64(e_o)
    if e.shape != (len(pairs),):
        raise ValueError("e_o must have one entry per pair")
    keep = np.zeros(len(pairs), dtype=np.uint8)
    _check(_lib.kvt_pareto_prune(_pairs(pairs), e.ctypes.data, len(pairs), keep.ctypes.data))
    return [bool(x) for x in keep]


def dbscan(points, eps: float = 0.05, min_samples: int = 2) -> list:
    """DBSCAN labels (cluster ids in order of discovery, -1 = noise) of points [n][dim] (App. D)."""
    import numpy as np
    x = _f64(points)
    if x.ndim != 2:
        raise ValueError("points must be [n][dim]")
    lab = np.zeros(x.shape[0], dtype=np.int32)
    _check(_lib.kvt_dbscan(x.ctypes.data, x.shape[0], x.shape[1], float(eps), int(min_samples), lab.ctypes.data))
    return [int(v) for v in lab]


def prune_and_cluster(pairs: Sequence[tuple], e_o, eps: float = 0.05, min_samples: int = 2):
    """Two-level search-space pruning: e_o [L][n_pairs] -> (keep [L][n_pairs] bool,
    group_of_layer [L], n_groups)."""
    import numpy as np
    e = _f64(e_o)
    if e.ndim != 2 or e.shape[1] != len(pairs):
        raise ValueError("e_o must be [n_layers][n_pairs]")
    L = e.shape[0]
    keep = np.zeros((L, len(pairs)), dtype=np.uint8)
    grp = np.zeros(L, dtype=np.int32)
    ng = ctypes.c_int32()
    _check(_lib.kvt_prune_and_cluster(_pairs(pairs), len(pairs), e.ctypes.data, L, float(eps), int(min_samples),
                                      keep.ctypes.data, grp.ctypes.data, ctypes.byref(ng)))
    return keep.astype(bool), [int(g) for g in grp], int(ng.value)


def search_space_log10(counts: Sequence[int]) -> float:
    """log10 of prod(counts): the search-space size S^L or S_p^G."""
    import numpy as np
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int32))
    out = ctypes.c_double()
    _check(_lib.kvt_search_space_log10(c.ctypes.data, c.size, ctypes.byref(out)))
    return float(out.value)
