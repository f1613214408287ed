"""CPU oracle for the FlexGen compressed-KV decode-attention hot path.

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs -- never by the
product package ``paper_2303_06865_b200``.  The arithmetic lives in
``flexq_oracle.c`` (plain C, built ``-O2 -ffp-contract=off``); this module is
ctypes marshalling over numpy arrays.  See flexq_oracle.c for the paper
passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "flexq_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]

_lib = None


def build(force: bool = False) -> str:
    """Compile flexq_oracle.c -> oracle/liboracle.so with gcc (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.oracle_f16_to_f32.argtypes = [ctypes.c_uint16]
        L.oracle_f16_to_f32.restype = ctypes.c_float
        L.oracle_f32_to_f16.argtypes = [ctypes.c_float]
        L.oracle_f32_to_f16.restype = ctypes.c_uint16
        L.oracle_quantize.argtypes = [P, i64, i64, i32, i32, P, P]
        L.oracle_pack4.argtypes = [P, i64, P]
        L.oracle_unpack4.argtypes = [P, i64, P]
        L.oracle_pack_bits.argtypes = [P, i64, i32, P]
        L.oracle_unpack_bits.argtypes = [P, i64, i32, P]
        L.oracle_dequantize.argtypes = [P, P, i64, i64, i32, i32, P]
        L.oracle_append_kv.argtypes = [P, P] + [i32] * 8 + [P, P, P, P]
        L.oracle_attention_f64.argtypes = [P] * 5 + [i32] * 6 + [P, P]
        L.oracle_attention_f32.argtypes = [P] * 5 + [i32] * 6 + [P]
        L.oracle_attention_topk_f64.argtypes = [P] * 5 + [i32] * 7 + [P, P, P, P]
        L.oracle_dequant_gemm_f64.argtypes = [P, P, P, i64, i64, i64, i32, i32, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def _h(a) -> np.ndarray:
    """fp16 array -> contiguous uint16 bit view."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float16:
        a = a.view(np.uint16)
    assert a.dtype == np.uint16
    return a


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"{what}: oracle status {rc}")


def f16_to_f32(bits: int) -> float:
    return lib().oracle_f16_to_f32(int(bits))


def f32_to_f16(x: float) -> int:
    return int(lib().oracle_f32_to_f16(float(np.float32(x))))


def quantize(x, bits: int = 4, group: int = 64):
    """x: fp16 [rows][cols] -> (codes u8 [rows][cols] unpacked, meta u16 [rows][cols/group][2])."""
    x = _h(x)
    rows, cols = x.shape
    codes = np.zeros((rows, cols), np.uint8)
    meta = np.zeros((rows, max(cols // group, 0), 2), np.uint16)
    _check(lib().oracle_quantize(_p(x), rows, cols, bits, group, _p(codes), _p(meta)), "quantize")
    return codes, meta


def pack4(codes: np.ndarray) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    out = np.zeros(codes.shape[:-1] + (codes.shape[-1] // 2,), np.uint8)
    _check(lib().oracle_pack4(_p(codes), codes.size, _p(out)), "pack4")
    return out


def unpack4(packed: np.ndarray) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    out = np.zeros(packed.shape[:-1] + (packed.shape[-1] * 2,), np.uint8)
    _check(lib().oracle_unpack4(_p(packed), out.size, _p(out)), "unpack4")
    return out


def pack_bits(codes: np.ndarray, bits: int) -> np.ndarray:
    """Little-endian bit stream of each row's codes: [..][n] -> [..][n * bits / 8] bytes."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n = codes.shape[-1]
    out = np.zeros(codes.shape[:-1] + (n * bits // 8,), np.uint8)
    rows = codes.reshape(-1, n)
    o = out.reshape(-1, n * bits // 8)
    for i in range(rows.shape[0]):
        r, oi = np.ascontiguousarray(rows[i]), np.zeros(n * bits // 8, np.uint8)
        _check(lib().oracle_pack_bits(_p(r), n, bits, _p(oi)), "pack_bits")
        o[i] = oi
    return out


def unpack_bits(packed: np.ndarray, n: int, bits: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    rows = packed.reshape(-1, packed.shape[-1])
    out = np.zeros((rows.shape[0], n), np.uint8)
    for i in range(rows.shape[0]):
        r, oi = np.ascontiguousarray(rows[i]), np.zeros(n, np.uint8)
        _check(lib().oracle_unpack_bits(_p(r), n, bits, _p(oi)), "unpack_bits")
        out[i] = oi
    return out.reshape(packed.shape[:-1] + (n,))


def dequantize(codes, meta, bits: int = 4, group: int = 64) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    meta = _h(meta)
    rows, cols = codes.shape
    out = np.zeros((rows, cols), np.uint16)
    _check(lib().oracle_dequantize(_p(codes), _p(meta), rows, cols, bits, group, _p(out)), "dequantize")
    return out.view(np.float16)


def empty_cache(B: int, H: int, T_cap: int, D: int, group: int = 64):
    """Oracle cache: codes u8 [B][H][T_cap][D] (unpacked), meta u16 [B][H][T_cap][D/group][2]."""
    return (np.zeros((B, H, T_cap, D), np.uint8), np.zeros((B, H, T_cap, D // group, 2), np.uint16))


def append_kv(k_new, v_new, k_cache, v_cache, pos: int, bits: int = 4, group: int = 64):
    """k_new, v_new: fp16 [B][H][n_new][D]; caches from empty_cache (modified in place)."""
    k_new, v_new = _h(k_new), _h(v_new)
    B, H, n_new, D = k_new.shape
    kc, km = k_cache
    vc, vm = v_cache
    T_cap = kc.shape[2]
    _check(lib().oracle_append_kv(_p(k_new), _p(v_new), B, H, D, T_cap, pos, n_new, bits, group,
                                  _p(kc), _p(km), _p(vc), _p(vm)), "append_kv")


def attention_f64(q, k_cache, v_cache, cur_len: int, group: int = 64,
                  want_probs: bool = False):
    """q: fp16 [B][H][D] -> out float64 [B][H][D] (and probs [B][H][cur_len] if asked)."""
    q = _h(q)
    B, H, D = q.shape
    kc, km = k_cache
    vc, vm = v_cache
    T_cap = kc.shape[2]
    out = np.zeros((B, H, D), np.float64)
    probs = np.zeros((B, H, cur_len), np.float64) if want_probs else None
    _check(lib().oracle_attention_f64(_p(q), _p(kc), _p(km), _p(vc), _p(vm), B, H, D, T_cap, cur_len,
                                      group, _p(out),
                                      _p(probs) if want_probs else None), "attention_f64")
    return (out, probs) if want_probs else out


def attention_f32(q, k_cache, v_cache, cur_len: int, group: int = 64):
    q = _h(q)
    B, H, D = q.shape
    kc, km = k_cache
    vc, vm = v_cache
    T_cap = kc.shape[2]
    out = np.zeros((B, H, D), np.float32)
    _check(lib().oracle_attention_f32(_p(q), _p(kc), _p(km), _p(vc), _p(vm), B, H, D, T_cap, cur_len,
                                      group, _p(out)), "attention_f32")
    return out


def attention_topk_f64(q, k_cache, v_cache, cur_len: int, keep: int, group: int = 64, sel=None):
    """Top-K sparse decode attention.
    -> (out float64 [B][H][D], kept mask u8 [B][H][cur_len], scores float64 [B][H][cur_len]).
    sel: optional kept mask to evaluate instead of selecting."""
    q = _h(q)
    B, H, D = q.shape
    kc, km = k_cache
    vc, vm = v_cache
    T_cap = kc.shape[2]
    out = np.zeros((B, H, D), np.float64)
    mask = np.zeros((B, H, cur_len), np.uint8)
    scores = np.zeros((B, H, cur_len), np.float64)
    sel_arr = None if sel is None else np.ascontiguousarray(sel, dtype=np.uint8)
    _check(lib().oracle_attention_topk_f64(_p(q), _p(kc), _p(km), _p(vc), _p(vm), B, H, D, T_cap, cur_len,
                                           group, keep, _p(sel_arr) if sel_arr is not None else None,
                                           _p(mask), _p(scores), _p(out)), "attention_topk_f64")
    return out, mask, scores


def dequant_gemm_f64(x, codes, meta, bits: int = 4, group: int = 64) -> np.ndarray:
    """Decode linear layer over a quantized weight.
    x: fp16 [M][K]; codes u8 [K][N] unpacked; meta u16 [K][N/group][2] -> float64 [M][N]."""
    x = _h(x)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    meta = _h(meta)
    M, K = x.shape
    K2, N = codes.shape
    assert K2 == K
    out = np.zeros((M, N), np.float64)
    _check(lib().oracle_dequant_gemm_f64(_p(x), _p(codes), _p(meta), M, K, N, bits, group, _p(out)),
           "dequant_gemm_f64")
    return out
