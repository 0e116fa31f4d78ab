"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of liboracle_ffa.so (ffa_oracle.c).

Callers: tests/, __graft_entry__.smoke(), bench.py (cpu_baseline and
--impl reference legs). The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_LIB = HERE / "liboracle_ffa.so"
_lib = None

_i64, _i32, _f64 = C.c_int64, C.c_int32, C.c_double
_P = C.c_void_p


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            build()
        L = C.CDLL(str(_LIB))
        L.oracle_ffa_fwd.argtypes = [_P, _P, _P, _i64, _i64, _i64, _i64, C.c_int, _P, _P, _P, _i64,
                                     _f64, _P, _P, C.c_int]
        L.oracle_ffa_fwd.restype = None
        L.oracle_ffa_bwd.argtypes = [_P, _P, _P, _P, _P, _P, _i64, _i64, _i64, _i64, C.c_int, _P, _P,
                                     _P, _i64, _f64, _P, _P, _P]
        L.oracle_ffa_bwd.restype = None
        L.oracle_num_threads.restype = C.c_int
        L.oracle_row_allowed.argtypes = [_i64, _i64, _i64, _i64, _i32, _i64, _i64]
        L.oracle_row_allowed.restype = C.c_int
        _lib = L
    return _lib


def _f32(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().float().cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float32)


def _slices(q_ranges, k_ranges, types):
    qr = np.ascontiguousarray(np.asarray(q_ranges, dtype=np.int64).reshape(-1, 2))
    kr = np.ascontiguousarray(np.asarray(k_ranges, dtype=np.int64).reshape(-1, 2))
    ty = np.ascontiguousarray(np.asarray(types, dtype=np.int32).reshape(-1))
    return qr, kr, ty


def num_threads() -> int:
    return lib().oracle_num_threads()


def ffa_fwd(q, k, v, q_ranges, k_ranges, types, scale, acc_f32=False):
    """q [sq, hq, d], k/v [sk, hk, d] (bf16-rounded values). Returns (out [sq,hq,d] f64, lse [hq,sq] f64)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    sq, hq, d = q.shape
    sk, hk, _ = k.shape
    qr, kr, ty = _slices(q_ranges, k_ranges, types)
    out = np.zeros((sq, hq, d), np.float64)
    lse = np.zeros((hq, sq), np.float64)
    lib().oracle_ffa_fwd(q.ctypes.data, k.ctypes.data, v.ctypes.data, sq, sk, hq, hk, d,
                         qr.ctypes.data, kr.ctypes.data, ty.ctypes.data, len(ty), float(scale),
                         out.ctypes.data, lse.ctypes.data, int(acc_f32))
    return out, lse


def ffa_bwd(q, k, v, out, lse, dout, q_ranges, k_ranges, types, scale):
    """Gradients in float64: (dq [sq,hq,d], dk [sk,hk,d], dv [sk,hk,d])."""
    q, k, v, dout = _f32(q), _f32(k), _f32(v), _f32(dout)
    out = np.ascontiguousarray(out, np.float64)
    lse = np.ascontiguousarray(lse, np.float64)
    sq, hq, d = q.shape
    sk, hk, _ = k.shape
    qr, kr, ty = _slices(q_ranges, k_ranges, types)
    dq = np.zeros((sq, hq, d), np.float64)
    dk = np.zeros((sk, hk, d), np.float64)
    dv = np.zeros((sk, hk, d), np.float64)
    lib().oracle_ffa_bwd(q.ctypes.data, k.ctypes.data, v.ctypes.data, out.ctypes.data,
                         lse.ctypes.data, dout.ctypes.data, sq, sk, hq, hk, d, qr.ctypes.data,
                         kr.ctypes.data, ty.ctypes.data, len(ty), float(scale), dq.ctypes.data,
                         dk.ctypes.data, dv.ctypes.data)
    return dq, dk, dv


def dense_allowed(sq, sk, q_ranges, k_ranges, types) -> np.ndarray:
    """Multiplicity count matrix [sq, sk] of the slice list (small cases only)."""
    qr, kr, ty = _slices(q_ranges, k_ranges, types)
    cnt = np.zeros((sq, sk), np.int32)
    L = lib()
    for (qs, qe), (ks, ke), t in zip(qr, kr, ty):
        for q in range(qs, qe):
            for kk in range(ks, ke):
                cnt[q, kk] += L.oracle_row_allowed(qs, qe, ks, ke, int(t), q, kk)
    return cnt
