"""CPU oracle for FastLSH hash evaluation — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and `--impl reference`)
may import this package. The product path (paper_2309_15479_b200/) never imports it and shares
no code with it.

Contents (each function cites the passage it follows):
  fastlsh_oracle.c  double-precision Eq. 5 / Eq. 1 evaluation
  brute.py          pure-Python triple loop for tiny inputs (must equal the C oracle bit for bit)
  keys.py           compound bucket keys with Python big integers (R9)
  theory.py         collision probabilities / moments used as statistical pins (PAPER.md:96-101,
                    184-269, 308-323)

Parity status: every function here is pinned by tests/test_oracle_pins.py (see DESIGN.md
"Oracle pins"); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fastlsh_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """gcc -O2 -fopenmp the oracle (no -ffast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
               "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
            _lib.oracle_hash.argtypes = [P, i64, i32, P, P, P, dbl, i32, i32, P, P, P, i32]
            _lib.oracle_hash.restype = None
            _lib.oracle_e2lsh.argtypes = [P, i64, i32, P, P, dbl, i32, P, P, P, i32]
            _lib.oracle_e2lsh.restype = None
            _lib.oracle_apply_sampling.argtypes = [P, i32, P, i32, P]
            _lib.oracle_apply_sampling.restype = None
            _lib.oracle_has_openmp.restype = ctypes.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def apply_sampling(v, idx):
    """S(v): out[j] = v[idx[j]]."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    out = np.empty(idx.shape[0], dtype=np.float64)
    lib().oracle_apply_sampling(_ptr(v), v.shape[0], _ptr(idx), idx.shape[0], _ptr(out))
    return out


def fastlsh(X, idx, a, b, w, threads: int = 1):
    """Eq. 5 for every row of X and every hash: returns (p f64[N,k], scale f64[N,k], code i64[N,k])."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    N, n = X.shape
    k, m = idx.shape
    assert a.shape == (k, m) and b.shape == (k,)
    if N and k:
        assert idx.min() >= 0 and idx.max() < n
    p = np.empty((N, k), np.float64)
    s = np.empty((N, k), np.float64)
    c = np.empty((N, k), np.int64)
    lib().oracle_hash(_ptr(X), N, n, _ptr(idx), _ptr(a), _ptr(b), float(w), k, m,
                      _ptr(p), _ptr(s), _ptr(c), int(threads))
    return p, s, c


def e2lsh(X, A, b, w, threads: int = 1):
    """Eq. 1 with dense A[k,n]: returns (p, scale, code)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    A = np.ascontiguousarray(A, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    N, n = X.shape
    k = A.shape[0]
    p = np.empty((N, k), np.float64)
    s = np.empty((N, k), np.float64)
    c = np.empty((N, k), np.int64)
    lib().oracle_e2lsh(_ptr(X), N, n, _ptr(A), _ptr(b), float(w), k, _ptr(p), _ptr(s), _ptr(c),
                       int(threads))
    return p, s, c


def has_openmp() -> bool:
    return bool(lib().oracle_has_openmp())
