"""CPU oracle for the KVTuner hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2502_04420_b200``) never imports it and shares no code with it.

The arithmetic lives in ``kvt_oracle.c`` (plain C, fp64 except where DESIGN.md fixes fp32),
each function citing the PAPER.md passage it follows; this module only marshals numpy arrays
through ctypes.  bf16 tensors are passed as ``uint16`` arrays holding the raw bf16 bits.

Parity status: every function here is pinned by ``tests/test_oracle_*.py`` (closed forms,
worked bytes, special cases, library routines) except the magnitudes of the O4 sensitivity
metrics on real LLM traces ("parity unpinned"): those need the paper's
Llama/Qwen GSM8K traces, which do not exist here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "kvt_oracle.c"
_LIB = _HERE / "libkvt_oracle.so"

MODE_PER_TOKEN = 0
MODE_KIVI = 1
MODE_PER_CHANNEL = 2        # sensitivity only (A28)
MODES = {"per-token-asym": MODE_PER_TOKEN, "kivi": MODE_KIVI, "per-channel-asym": MODE_PER_CHANNEL}


def build(force: bool = False) -> Path:
    """Compile the oracle (gcc, -O2 -ffp-contract=off: IEEE fp32 order, no FMA contraction)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < max(_SRC.stat().st_mtime,
                                                                 (_HERE / "kvt_oracle.h").stat().st_mtime):
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
        P = ctypes.c_void_p
        i = ctypes.c_int
        _lib.kvto_bf16_to_f32.restype = ctypes.c_float
        _lib.kvto_bf16_to_f32.argtypes = [ctypes.c_uint16]
        _lib.kvto_f32_to_bf16_rne.restype = ctypes.c_uint16
        _lib.kvto_f32_to_bf16_rne.argtypes = [ctypes.c_float]
        _lib.kvto_f32_to_bf16_ru.restype = ctypes.c_uint16
        _lib.kvto_f32_to_bf16_ru.argtypes = [ctypes.c_float]
        _lib.kvto_quantize_group.argtypes = [P, i, i, i, P, P]
        _lib.kvto_dequant_value.restype = ctypes.c_double
        _lib.kvto_dequant_value.argtypes = [ctypes.c_uint8, ctypes.c_uint32]
        _lib.kvto_pack_row.argtypes = [P, i, i, P]
        _lib.kvto_unpack_row.argtypes = [P, i, i, P]
        _lib.kvto_n_quantized_key.argtypes = [i, i, i, i, i]
        _lib.kvto_n_quantized_value.argtypes = [i, i, i, i, i]
        _lib.kvto_slice_bytes.argtypes = [i, i, i, i, i, i, i, P]
        _lib.kvto_build_cache.argtypes = [i, i, i, i, i, i, i, i, P, P, P, P, P, P, P, P]
        _lib.kvto_dequant_cache.argtypes = [i, i, i, i, i, i, i, i, P, P, P, P, P, P, P, P]
        _lib.kvto_attention.argtypes = [P, i, P, P, i, i, ctypes.c_double, P, P]
        _lib.kvto_sensitivity.argtypes = [i, i, i, P, i, i, i, P, P, i, i, i, ctypes.c_double, P, i, P]
        _lib.kvto_layer_decode.argtypes = [i, i, i, i, i, i, i, i, i, i, P, P, P, P, ctypes.c_double, P]
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _u16(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    assert a.dtype == np.uint16, f"expected raw bf16 bits as uint16, got {a.dtype}"
    return a


# ---------------------------------------------------------------------------------------------
# scalar bf16 helpers
# ---------------------------------------------------------------------------------------------
def bf16_to_f32(bits: int) -> float:
    return float(lib().kvto_bf16_to_f32(int(bits)))


def f32_to_bf16_rne(x: float) -> int:
    return int(lib().kvto_f32_to_bf16_rne(float(x)))


def f32_to_bf16_ru(x: float) -> int:
    return int(lib().kvto_f32_to_bf16_ru(float(x)))


def bf16_array_to_f64(a: np.ndarray) -> np.ndarray:
    """Widen raw bf16 bits to fp64 (exact)."""
    return (np.asarray(a, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------------------------
# O1
# ---------------------------------------------------------------------------------------------
def quantize_group(x_bf16: np.ndarray, bits: int):
    """O1 on one group: returns (codes uint8[n], meta uint32)."""
    x = _u16(x_bf16).reshape(-1)
    codes = np.zeros(x.size, np.uint8)
    meta = np.zeros(1, np.uint32)
    lib().kvto_quantize_group(_p(x), x.size, 1, bits, _p(codes), _p(meta))
    return codes, int(meta[0])


def dequant_value(code: int, meta: int) -> float:
    return float(lib().kvto_dequant_value(code, meta))


def meta_scale_zero(meta: int):
    """(scale, zero) as floats from a meta word (low 16 bits scale, high 16 bits zero)."""
    return bf16_to_f32(meta & 0xFFFF), bf16_to_f32(meta >> 16)


def pack_row(codes: np.ndarray, bits: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    row = np.zeros(codes.size * bits // 8, np.uint8)
    lib().kvto_pack_row(_p(codes), codes.size, bits, _p(row))
    return row


def unpack_row(row: np.ndarray, d: int, bits: int) -> np.ndarray:
    row = np.ascontiguousarray(row, dtype=np.uint8)
    codes = np.zeros(d, np.uint8)
    lib().kvto_unpack_row(_p(row), d, bits, _p(codes))
    return codes


# ---------------------------------------------------------------------------------------------
# O2
# ---------------------------------------------------------------------------------------------
def n_quantized_key(mode: int, bits: int, G: int, R: int, S: int) -> int:
    return int(lib().kvto_n_quantized_key(mode, bits, G, R, S))


def n_quantized_value(mode: int, bits: int, G: int, R: int, S: int) -> int:
    return int(lib().kvto_n_quantized_value(mode, bits, G, R, S))


def slice_bytes(mode: int, kb: int, vb: int, G: int, R: int, d: int, cap: int):
    out = np.zeros(6, np.uint64)
    rc = lib().kvto_slice_bytes(mode, kb, vb, G, R, d, cap, _p(out))
    if rc != 0:
        raise ValueError("invalid cache geometry")
    return [int(v) for v in out]


BUFFER_NAMES = ("k_codes", "k_meta", "k_resid", "v_codes", "v_meta", "v_resid")
_BUF_DTYPES = (np.uint8, np.uint32, np.uint16, np.uint8, np.uint32, np.uint16)


def build_cache(mode, kb, vb, G, R, d, cap, K_bf16, V_bf16, fill=0):
    """O2 for one (b, h) slice: K, V uint16 [S][d] → dict of the six buffers (numpy).  Bytes the
    layout does not define for this history keep the value `fill` (build twice with different fills
    to get the mask of defined bytes)."""
    K = _u16(K_bf16).reshape(-1, d)
    V = _u16(V_bf16).reshape(-1, d)
    S = K.shape[0]
    assert V.shape[0] == S
    sz = slice_bytes(mode, kb, vb, G, R, d, cap)
    bufs = [np.full(max(n // np.dtype(t).itemsize, 1), 0, t) for n, t in zip(sz, _BUF_DTYPES)]
    for b in bufs:
        b.view(np.uint8)[:] = fill
    rc = lib().kvto_build_cache(mode, kb, vb, G, R, d, cap, S, _p(K), _p(V), *[_p(b) for b in bufs])
    if rc != 0:
        raise ValueError("kvto_build_cache rejected its arguments")
    return dict(zip(BUFFER_NAMES, bufs))


def defined_bytes(mode, kb, vb, G, R, d, cap, K_bf16, V_bf16):
    """(bytes, mask) per buffer: the oracle's bytes and which of them the layout defines for this
    history (those identical under two different fill values)."""
    a = build_cache(mode, kb, vb, G, R, d, cap, K_bf16, V_bf16, fill=0x00)
    b = build_cache(mode, kb, vb, G, R, d, cap, K_bf16, V_bf16, fill=0xFF)
    return {n: (a[n].view(np.uint8), a[n].view(np.uint8) == b[n].view(np.uint8)) for n in BUFFER_NAMES}


def dequant_cache(mode, kb, vb, G, R, d, cap, S, bufs):
    """Read K_hat, V_hat [S][d] fp64 back from one (b, h) slice of buffers."""
    Kh = np.zeros((max(S, 1), d), np.float64)
    Vh = np.zeros((max(S, 1), d), np.float64)
    arrs = [np.ascontiguousarray(bufs[n], dtype=t) for n, t in zip(BUFFER_NAMES, _BUF_DTYPES)]
    rc = lib().kvto_dequant_cache(mode, kb, vb, G, R, d, cap, S, *[_p(a) for a in arrs], _p(Kh), _p(Vh))
    if rc != 0:
        raise ValueError("kvto_dequant_cache rejected its arguments")
    return Kh[:S], Vh[:S]


# ---------------------------------------------------------------------------------------------
# O3
# ---------------------------------------------------------------------------------------------
def attention(q_bf16: np.ndarray, Khat: np.ndarray, Vhat: np.ndarray, scale: float, with_probs=False):
    """Eq. 1 in fp64.  q uint16 [g][d]; Khat/Vhat fp64 [S][d] → out fp64 [g][d] (and probs [g][S])."""
    q = _u16(q_bf16)
    d = q.shape[-1]
    q = q.reshape(-1, d)
    g = q.shape[0]
    Kh = np.ascontiguousarray(Khat, dtype=np.float64).reshape(-1, d)
    Vh = np.ascontiguousarray(Vhat, dtype=np.float64).reshape(-1, d)
    S = Kh.shape[0]
    out = np.zeros((g, d), np.float64)
    probs = np.zeros((g, max(S, 1)), np.float64) if with_probs else None
    lib().kvto_attention(_p(q), g, _p(Kh), _p(Vh), S, d, float(scale), _p(out),
                         _p(probs) if with_probs else None)
    return (out, probs[:, :S]) if with_probs else out


def decode_reference(mode, kb, vb, G, R, d, K_bf16, V_bf16, q_bf16, scale):
    """O2 + O3 for one (b, kv head): the expected fp64 output [g][d] for a cache holding K, V."""
    S = _u16(K_bf16).reshape(-1, d).shape[0]
    cap = max(((S + G - 1) // G) * G, G)
    bufs = build_cache(mode, kb, vb, G, R, d, cap, K_bf16, V_bf16)
    Kh, Vh = dequant_cache(mode, kb, vb, G, R, d, cap, S, bufs)
    return attention(q_bf16, Kh, Vh, scale)


def layer_decode(mode, kb, vb, G, R, K_bf16, V_bf16, q_bf16, seq_len, scale):
    """Whole layer: K, V uint16 [B][H_kv][S_max][d]; q uint16 [B][H_q][d] → fp64 [B][H_q][d]."""
    K = _u16(K_bf16)
    V = _u16(V_bf16)
    q = _u16(q_bf16)
    B, H_kv, S_max, d = K.shape
    H_q = q.shape[1]
    sl = np.ascontiguousarray(seq_len, dtype=np.int32)
    out = np.zeros((B, H_q, d), np.float64)
    rc = lib().kvto_layer_decode(mode, kb, vb, G, R, B, H_kv, H_q, d, S_max, _p(sl), _p(K), _p(V), _p(q),
                                 float(scale), _p(out))
    if rc != 0:
        raise ValueError("kvto_layer_decode rejected its arguments")
    return out


# ---------------------------------------------------------------------------------------------
# O4
# ---------------------------------------------------------------------------------------------
ERROR_NAMES = ("e_k", "e_v", "e_a", "e_o", "e_o_l1")


def sensitivity(mode, G, R, Q_bf16, K_bf16, V_bf16, q_pos0, pairs, scale):
    """Q uint16 [H_q][T_q][d]; K, V uint16 [H_kv][S][d]; pairs [(b_k, b_v), ...] → fp64 [n_pairs][5]."""
    Q = _u16(Q_bf16)
    K = _u16(K_bf16)
    V = _u16(V_bf16)
    H_q, T_q, d = Q.shape
    H_kv, S, _ = K.shape
    pb = np.ascontiguousarray(np.array(pairs, dtype=np.int32).reshape(-1, 2))
    out = np.zeros((pb.shape[0], 5), np.float64)
    rc = lib().kvto_sensitivity(mode, G, R, _p(Q), H_q, T_q, q_pos0, _p(K), _p(V), H_kv, S, d, float(scale),
                                _p(pb), pb.shape[0], _p(out))
    if rc != 0:
        raise ValueError("kvto_sensitivity rejected its arguments")
    return out
