"""paper_2309_15479_b200 — FastLSH hash evaluation on B200 (sm_100a).

Thin ctypes binding over libfastlsh.so (include/fastlsh.h). Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels; torch supplies device memory and streams.
There is no CPU fallback: if the library is missing or the device is not a B200, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfastlsh.so")

OK, EINVAL, ENOMEM, ECUDA, EUNSUPPORTED, ESTATE = 0, -1, -2, -3, -4, -5

EXPORTED = [
    "fastlsh_params_create", "fastlsh_params_create_from_arrays", "e2lsh_params_create",
    "fastlsh_params_destroy", "fastlsh_params_export", "fastlsh_params_info", "fastlsh_params_packing",
    "fastlsh_params_row_packing",
    "fastlsh_params_upload", "fastlsh_params_set_kernel", "fastlsh_params_set_table_size",
    "fastlsh_params_prepare", "fastlsh_params_jit_status", "fastlsh_params_jit_check",
    "fastlsh_hash", "fastlsh_project", "e2lsh_hash", "e2lsh_project", "fastlsh_keys_create",
    "fastlsh_keys_create_from_arrays", "fastlsh_keys_destroy", "fastlsh_keys_export",
    "fastlsh_build_keys", "fastlsh_hash_keys", "fastlsh_hash_keys_multicast", "fastlsh_tables_workspace",
    "fastlsh_build_tables",
    "fastlsh_query_workspace", "fastlsh_query", "fastlsh_normalize_rows", "fastlsh_max_row_norm",
    "fastlsh_mips_transform", "fastlsh_hash_host", "fastlsh_read_flags",
    "fastlsh_bandwidth_probe", "fastlsh_multicast_alloc", "fastlsh_multicast_free", "fastlsh_status_string", "fastlsh_last_cuda_error", "fastlsh_abi_version",
]


class FastLSHError(RuntimeError):
    def __init__(self, status: int, what: str):
        lib = _lib
        msg = lib.fastlsh_status_string(status).decode() if lib else str(status)
        if status == ECUDA and lib:
            msg += f" ({lib.fastlsh_last_cuda_error().decode()})"
        super().__init__(f"{what}: {msg} [{status}]")
        self.status = status


class _Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("k", ctypes.c_int32),
                ("w", ctypes.c_float), ("is_e2lsh", ctypes.c_int32), ("parts", ctypes.c_int32),
                ("slots", ctypes.c_int32), ("units", ctypes.c_int32),
                ("warps_per_block", ctypes.c_int32), ("hash_blocks", ctypes.c_int32),
                ("rows_per_group", ctypes.c_int32), ("bank_efficiency", ctypes.c_double),
                ("conflict_wavefronts", ctypes.c_int64), ("kernel", ctypes.c_int32),
                ("tmem_hash_blocks", ctypes.c_int32), ("tmem_hashes_per_warp", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libfastlsh.so (build it with __graft_entry__.build() or paper_2309_15479_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libfastlsh.so not built at {path}; run `python __graft_entry__.py build`")
    lib = ctypes.CDLL(path)
    P, i32, i64, u64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "fastlsh_params_create": [i32, i32, i32, f32, u64, PP],
        "fastlsh_params_create_from_arrays": [i32, i32, i32, f32, P, P, P, PP],
        "e2lsh_params_create": [i32, i32, f32, u64, PP],
        "fastlsh_params_export": [P, P, P, P, P],
        "fastlsh_params_info": [P, ctypes.POINTER(_Info)],
        "fastlsh_params_upload": [P, i32, P],
        "fastlsh_params_set_kernel": [P, i32],
        "fastlsh_params_set_table_size": [P, i32],
        "fastlsh_params_prepare": [P, P, i32],
        "fastlsh_params_jit_status": [P, ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, i64],
        "fastlsh_params_jit_check": [P, P, i32, ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, i64],
        "fastlsh_params_packing": [P, P, P, P, P, P, P],
        "fastlsh_params_row_packing": [P, P, P, P, P, P, P],
        "fastlsh_hash": [P, P, i64, P, P],
        "fastlsh_project": [P, P, i64, P, P],
        "e2lsh_hash": [P, P, i64, P, i32, P],
        "e2lsh_project": [P, P, i64, P, i32, P],
        "fastlsh_keys_create": [i32, i32, u64, PP],
        "fastlsh_keys_create_from_arrays": [i32, i32, P, PP],
        "fastlsh_keys_export": [P, P],
        "fastlsh_build_keys": [P, P, i64, i32, P, i64, P],
        "fastlsh_hash_keys": [P, P, P, i64, P, P, i64, P],
        "fastlsh_hash_keys_multicast": [P, P, P, i64, P, P, i64, P],
        "fastlsh_tables_workspace": [i32, i64, ctypes.POINTER(ctypes.c_size_t)],
        "fastlsh_build_tables": [P, i32, i64, i64, P, P, P, P, P, ctypes.c_size_t, P],
        "fastlsh_query_workspace": [i64, i64, ctypes.POINTER(ctypes.c_size_t)],
        "fastlsh_normalize_rows": [P, i64, i32, P, P],
        "fastlsh_max_row_norm": [P, i64, i32, P, P],
        "fastlsh_mips_transform": [P, i64, i32, P, i32, P, P],
        "fastlsh_query": [P, i64, i32, P, P, i32, P, P, i64, i64, i32, P, P, P, P, ctypes.c_size_t, P],
        "fastlsh_hash_host": [P, P, P, i64, P, P, i64],
        "fastlsh_read_flags": [P, P, P, i32, P],
        "fastlsh_bandwidth_probe": [P, P, i64, i32, i32, P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.fastlsh_multicast_alloc.argtypes = [ctypes.c_size_t, PP, PP, PP]
    lib.fastlsh_multicast_alloc.restype = ctypes.c_int
    lib.fastlsh_multicast_free.argtypes = [P]
    lib.fastlsh_multicast_free.restype = None
    lib.fastlsh_params_destroy.argtypes = [P]
    lib.fastlsh_params_destroy.restype = None
    lib.fastlsh_keys_destroy.argtypes = [P]
    lib.fastlsh_keys_destroy.restype = None
    lib.fastlsh_status_string.argtypes = [ctypes.c_int]
    lib.fastlsh_status_string.restype = ctypes.c_char_p
    lib.fastlsh_last_cuda_error.restype = ctypes.c_char_p
    lib.fastlsh_abi_version.restype = ctypes.c_int32
    _lib = lib
    return lib


def _check(status: int, what: str):
    if status != OK:
        raise FastLSHError(status, what)


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dev_ptr(t, dtype, what: str):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA torch tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{what} must be a contiguous {dtype} tensor")
    return ctypes.c_void_p(t.data_ptr())


def _check_X(params, X, what: str = "X"):
    if X.ndim != 2 or X.shape[1] != params.n:
        raise ValueError(f"{what} must be [N, n={params.n}], got {tuple(X.shape)}")


def _check_out(out, rows: int, cols: int, what: str):
    if out.ndim != 2 or tuple(out.shape) != (rows, cols):
        raise ValueError(f"{what} must be [{rows}, {cols}], got {tuple(out.shape)}")


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Params:
    """FastLSH (or E2LSH) hash-function parameters: S_i, a_i, b_i, w."""

    def __init__(self, handle: int, lib):
        self._h = ctypes.c_void_p(handle)
        self._lib = lib
        info = self.info()
        self.n, self.m, self.k, self.w = info["n"], info["m"], info["k"], info["w"]
        self._uploaded = set()

    @classmethod
    def create(cls, n: int, m: int, k: int, w: float, seed: int):
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.fastlsh_params_create(n, m, k, w, seed, ctypes.byref(h)), "fastlsh_params_create")
        return cls(h.value, lib)

    @classmethod
    def from_arrays(cls, n: int, w: float, idx, a, b):
        lib = load_library()
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        k, m = idx.shape
        h = ctypes.c_void_p()
        _check(lib.fastlsh_params_create_from_arrays(n, m, k, w, _np_ptr(idx), _np_ptr(a), _np_ptr(b),
                                                     ctypes.byref(h)), "fastlsh_params_create_from_arrays")
        return cls(h.value, lib)

    @classmethod
    def e2lsh(cls, n: int, k: int, w: float, seed: int):
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.e2lsh_params_create(n, k, w, seed, ctypes.byref(h)), "e2lsh_params_create")
        return cls(h.value, lib)

    def info(self) -> dict:
        inf = _Info()
        _check(self._lib.fastlsh_params_info(self._h, ctypes.byref(inf)), "fastlsh_params_info")
        return {f: getattr(inf, f) for f, _ in _Info._fields_}

    def export(self):
        idx = np.empty((self.k, self.m), np.int32)
        a = np.empty((self.k, self.m), np.float32)
        b = np.empty(self.k, np.float32)
        w = ctypes.c_float()
        _check(self._lib.fastlsh_params_export(self._h, _np_ptr(idx), _np_ptr(a), _np_ptr(b), ctypes.byref(w)),
               "fastlsh_params_export")
        return idx, a, b, w.value

    def packing(self) -> dict:
        """The bank-scheduled GPU layout (diagnostic; see fastlsh_params_packing)."""
        sz = np.zeros(8, np.int32)
        _check(self._lib.fastlsh_params_packing(self._h, _np_ptr(sz), None, None, None, None, None),
               "fastlsh_params_packing")
        P, MS, W, HB, kbm, nq, sc, lanes = (int(x) for x in sz)
        offp = np.zeros(HB * W * MS * 32, np.uint32)
        coef = np.zeros(HB * W * MS * 32, np.float32)
        unit = np.zeros(HB * kbm * P, np.uint16)
        h0 = np.zeros(HB, np.int32)
        kb = np.zeros(HB, np.int32)
        _check(self._lib.fastlsh_params_packing(self._h, _np_ptr(sz), _np_ptr(offp), _np_ptr(coef), _np_ptr(unit),
                                                _np_ptr(h0), _np_ptr(kb)), "fastlsh_params_packing")
        return dict(parts=P, slots=MS, warps=W, hash_blocks=HB, kb_max=kbm, nq=nq, stage_chunks=sc,
                    offp=offp.reshape(HB, W, MS, 32), coef=coef.reshape(HB, W, MS, 32),
                    unit_lane=unit.reshape(HB, kbm, P), block_h0=h0, block_kb=kb)

    def row_packing(self) -> dict | None:
        """The K1r layout (diagnostic; see fastlsh_params_row_packing); None when K1r does not apply."""
        sz = np.zeros(10, np.int32)
        _check(self._lib.fastlsh_params_row_packing(self._h, _np_ptr(sz), None, None, None, None, None),
               "fastlsh_params_row_packing")
        ok, P, MS, W, HB, kbm, S, conf, S0, n1 = (int(x) for x in sz)
        if not ok:
            return None
        offp = np.zeros(HB * W * (MS // 2) * 32, np.uint32)
        coef = np.zeros(HB * W * MS * 32, np.float32)
        lh = np.zeros(HB * W * 32, np.int16)
        h0 = np.zeros(HB, np.int32)
        kb = np.zeros(HB, np.int32)
        _check(self._lib.fastlsh_params_row_packing(self._h, _np_ptr(sz), _np_ptr(offp), _np_ptr(coef), _np_ptr(lh),
                                                    _np_ptr(h0), _np_ptr(kb)), "fastlsh_params_row_packing")
        return dict(parts=P, slots=MS, warps=W, hash_blocks=HB, kb_max=kbm, S=S, conflicts=conf, S0=S0, n1=n1,
                    offp=offp.reshape(HB, W, MS // 2, 32), coef=coef.reshape(HB, W, MS, 32),
                    lane_hash=lh.reshape(HB, W, 32), block_h0=h0, block_kb=kb)

    KERNELS = {0: "K0", 1: "K1", 2: "K1t", 3: "K1r", 4: "K1j", 5: "K4 dense"}

    def set_kernel(self, kernel):
        """Pin the hashing kernel: "auto" (0), "smem" (1, K1), "tmem" (2, K1t), "rows" (3, K1r),
        "jit" (4, K1j) or "dense" (5, K4 on the merged coefficients); see fastlsh_params_set_kernel.
        Returns self."""
        code = {"auto": 0, "smem": 1, "tmem": 2, "rows": 3, "jit": 4, "dense": 5}.get(kernel, kernel)
        _check(self._lib.fastlsh_params_set_kernel(self._h, int(code)), "fastlsh_params_set_kernel")
        return self

    def prepare(self, keys=None, codes: bool = True, proj: bool = False):
        """K1j: compile the kernel variants later calls will use (fastlsh_params_prepare), so the
        first hash call does not pay the NVRTC compile. No-op for params served by K1r / K1."""
        what = (1 if codes else 0) | (2 if proj else 0) | (4 if keys is not None else 0)
        _check(self._lib.fastlsh_params_prepare(self._h, keys._h if keys is not None else None, what),
               "fastlsh_params_prepare")
        return self

    def jit_status(self) -> dict:
        """K1j diagnostics: NVRTC seconds spent so far and the last compile/load error."""
        sec = ctypes.c_double()
        buf = ctypes.create_string_buffer(4096)
        _check(self._lib.fastlsh_params_jit_status(self._h, ctypes.byref(sec), buf, len(buf)),
               "fastlsh_params_jit_status")
        return {"compile_seconds": sec.value, "error": buf.value.decode(errors="replace")}

    def jit_check(self, keys=None, what: int = 0b11) -> float:
        """K1j: generate + compile (no load, no GPU needed) the variants in `what` (bit 0 codes,
        1 projections, 2 codes + keys, 3 keys only, 4 multicast keys); returns NVRTC seconds."""
        sec = ctypes.c_double()
        buf = ctypes.create_string_buffer(4096)
        st = self._lib.fastlsh_params_jit_check(self._h, keys._h if keys is not None else None, int(what),
                                                ctypes.byref(sec), buf, len(buf))
        if st != OK:
            raise FastLSHError(st, "fastlsh_params_jit_check: " + buf.value.decode(errors="replace")[:500])
        return sec.value

    def set_table_size(self, K: int):
        """Pack hash blocks as whole tables of K hashes so keys are built inside the hashing kernel
        (fastlsh_params_set_table_size); call before the first upload."""
        _check(self._lib.fastlsh_params_set_table_size(self._h, int(K)), "fastlsh_params_set_table_size")
        return self

    def upload(self, device=None, stream=None):
        import torch
        dev = torch.cuda.current_device() if device is None else int(device)
        if dev in self._uploaded:
            return self
        with torch.cuda.device(dev):
            _check(self._lib.fastlsh_params_upload(self._h, dev, _stream_ptr(stream)), "fastlsh_params_upload")
        self._uploaded.add(dev)
        return self

    def _ready(self):
        import torch
        if torch.cuda.current_device() not in self._uploaded:
            self.upload()

    def close(self):
        if self._h is not None and self._h.value:
            self._lib.fastlsh_params_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Keys:
    """Compound-key multipliers r[L][K+1] (reading R9)."""

    def __init__(self, handle: int, lib, L: int, K: int):
        self._h = ctypes.c_void_p(handle)
        self._lib = lib
        self.L, self.K = L, K

    @classmethod
    def create(cls, L: int, K: int, seed: int):
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.fastlsh_keys_create(L, K, seed, ctypes.byref(h)), "fastlsh_keys_create")
        return cls(h.value, lib, L, K)

    @classmethod
    def from_arrays(cls, r):
        lib = load_library()
        r = np.ascontiguousarray(r, dtype=np.uint64)
        L, K1 = r.shape
        h = ctypes.c_void_p()
        _check(lib.fastlsh_keys_create_from_arrays(L, K1 - 1, _np_ptr(r), ctypes.byref(h)),
               "fastlsh_keys_create_from_arrays")
        return cls(h.value, lib, L, K1 - 1)

    def export(self):
        r = np.empty((self.L, self.K + 1), np.uint64)
        _check(self._lib.fastlsh_keys_export(self._h, _np_ptr(r)), "fastlsh_keys_export")
        return r

    def close(self):
        if self._h is not None and self._h.value:
            self._lib.fastlsh_keys_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fastlsh_hash(params: Params, X, out=None, stream=None):
    """codes[N,k] int32 = floor((a_i . S_i(x) + b_i) / w) (Eq. 5) for X f32 [N,n] on the GPU."""
    import torch
    params._ready()
    _check_X(params, X)
    N = X.shape[0]
    if out is None:
        out = torch.empty((N, params.k), dtype=torch.int32, device=X.device)
    _check_out(out, N, params.k, "codes")
    _check(params._lib.fastlsh_hash(params._h, _dev_ptr(X, torch.float32, "X"), N,
                                    _dev_ptr(out, torch.int32, "codes"), _stream_ptr(stream)), "fastlsh_hash")
    return out


def fastlsh_project(params: Params, X, out=None, stream=None):
    """proj[N,k] f32 = a_i . S_i(x) — the projection before +b, /w, floor."""
    import torch
    params._ready()
    _check_X(params, X)
    N = X.shape[0]
    if out is None:
        out = torch.empty((N, params.k), dtype=torch.float32, device=X.device)
    _check_out(out, N, params.k, "proj")
    _check(params._lib.fastlsh_project(params._h, _dev_ptr(X, torch.float32, "X"), N,
                                       _dev_ptr(out, torch.float32, "proj"), _stream_ptr(stream)), "fastlsh_project")
    return out


def e2lsh_hash(params: Params, X, out=None, precision: int = 3, stream=None):
    """Dense baseline codes on tcgen05: precision 3 = 3xTF32 (default), 2 = 3xFP16, 1 = plain TF32."""
    import torch
    params._ready()
    _check_X(params, X)
    N = X.shape[0]
    if out is None:
        out = torch.empty((N, params.k), dtype=torch.int32, device=X.device)
    _check_out(out, N, params.k, "codes")
    _check(params._lib.e2lsh_hash(params._h, _dev_ptr(X, torch.float32, "X"), N,
                                  _dev_ptr(out, torch.int32, "codes"), precision, _stream_ptr(stream)), "e2lsh_hash")
    return out


def e2lsh_project(params: Params, X, out=None, precision: int = 3, stream=None):
    import torch
    params._ready()
    _check_X(params, X)
    N = X.shape[0]
    if out is None:
        out = torch.empty((N, params.k), dtype=torch.float32, device=X.device)
    _check_out(out, N, params.k, "proj")
    _check(params._lib.e2lsh_project(params._h, _dev_ptr(X, torch.float32, "X"), N,
                                     _dev_ptr(out, torch.float32, "proj"), precision, _stream_ptr(stream)),
           "e2lsh_project")
    return out


def build_keys(keys: Keys, codes, out=None, ldk=None, stream=None, col0: int = 0):
    """keys[L, N] uint64 (stored in an int64 tensor) from codes[N, k] int32.

    With `out` an [L, ldk] tensor and `col0` > 0, the N keys of each table go to columns
    [col0, col0 + N) (chunked table builds)."""
    import torch
    if codes.ndim != 2:
        raise ValueError(f"codes must be [N, k], got {tuple(codes.shape)}")
    N, k = codes.shape
    if keys.L * keys.K > k:
        raise ValueError(f"codes has k={k} < L*K={keys.L * keys.K}")
    if out is None:
        ldk = (N + col0) if ldk is None else ldk
        out = torch.empty((keys.L, ldk), dtype=torch.int64, device=codes.device)
    ldk = out.shape[1]
    if out.shape[0] != keys.L or col0 < 0 or col0 + N > ldk:
        raise ValueError("keys output must be [L, ldk] with col0 + N <= ldk")
    ptr = ctypes.c_void_p(_dev_ptr(out, torch.int64, "keys").value + 8 * col0)
    _check(keys._lib.fastlsh_build_keys(keys._h, _dev_ptr(codes, torch.int32, "codes"), N, k, ptr, ldk,
                                        _stream_ptr(stream)), "fastlsh_build_keys")
    return out


def build_tables(keys, N=None, out=None, workspace=None, stream=None):
    """Bucket tables from keys [L, ldk] (int64 view of u64), rows [0, N).

    Returns (sorted_keys int64 [L, N], ids int32 [L, N] (u32 bit patterns), bucket_start int32
    [L, N+1], nbuckets int64 [L]); see fastlsh_build_tables."""
    import torch
    lib = load_library()
    L, ldk = keys.shape
    N = ldk if N is None else N
    dev = keys.device
    if out is None:
        out = (torch.empty((L, N), dtype=torch.int64, device=dev), torch.empty((L, N), dtype=torch.int32, device=dev),
               torch.empty((L, N + 1), dtype=torch.int32, device=dev), torch.empty((L,), dtype=torch.int64, device=dev))
    sk, ids, starts, nb = out
    need = ctypes.c_size_t()
    _check(lib.fastlsh_tables_workspace(L, N, ctypes.byref(need)), "fastlsh_tables_workspace")
    if workspace is None or workspace.numel() < need.value:
        workspace = torch.empty((max(1, need.value),), dtype=torch.uint8, device=dev)
    _check(lib.fastlsh_build_tables(_dev_ptr(keys, torch.int64, "keys"), L, N, ldk,
                                    _dev_ptr(sk, torch.int64, "sorted_keys") if N else None,
                                    _dev_ptr(ids, torch.int32, "ids") if N else None,
                                    _dev_ptr(starts, torch.int32, "bucket_start"), _dev_ptr(nb, torch.int64, "nbuckets"),
                                    ctypes.c_void_p(workspace.data_ptr()), workspace.numel(), _stream_ptr(stream)),
           "fastlsh_build_tables")
    return sk, ids, starts, nb


def query(X, tables, Q, qkeys, topk: int = 10, workspace=None, stream=None):
    """LSH query with exact re-ranking: tables = build_tables(...) output for X,
    qkeys [L, >= nq] the queries' keys. Returns (ids int32 [nq, topk], dist f32 [nq, topk],
    ncand int64 [nq])."""
    import torch
    lib = load_library()
    sk, ids, _starts, _nb = tables
    N, n = X.shape
    nq = Q.shape[0]
    L, ldq = qkeys.shape
    if Q.ndim != 2 or Q.shape[1] != n:
        raise ValueError(f"Q must be [nq, n={n}], got {tuple(Q.shape)}")
    if sk.shape[0] != L or ids.shape[0] != L or sk.shape[1] != N or ids.shape[1] != N:
        raise ValueError(f"tables must be [L={L}, N={N}] (the L of qkeys and the rows of X)")
    if ldq < nq:
        raise ValueError(f"qkeys must have >= nq={nq} columns")
    dev = Q.device
    out_i = torch.empty((nq, topk), dtype=torch.int32, device=dev)
    out_d = torch.empty((nq, topk), dtype=torch.float32, device=dev)
    out_c = torch.empty((nq,), dtype=torch.int64, device=dev)
    need = ctypes.c_size_t()
    _check(lib.fastlsh_query_workspace(N, nq, ctypes.byref(need)), "fastlsh_query_workspace")
    if workspace is None or workspace.numel() < need.value:
        workspace = torch.empty((max(1, need.value),), dtype=torch.uint8, device=dev)
    _check(lib.fastlsh_query(_dev_ptr(X, torch.float32, "X"), N, n, _dev_ptr(sk, torch.int64, "sorted_keys"),
                             _dev_ptr(ids, torch.int32, "ids"), L, _dev_ptr(Q, torch.float32, "Q"),
                             _dev_ptr(qkeys, torch.int64, "qkeys"), nq, ldq, topk,
                             _dev_ptr(out_i, torch.int32, "out_ids"), _dev_ptr(out_d, torch.float32, "out_dist"),
                             _dev_ptr(out_c, torch.int64, "out_ncand"), ctypes.c_void_p(workspace.data_ptr()),
                             workspace.numel(), _stream_ptr(stream)), "fastlsh_query")
    return out_i, out_d, out_c


def normalize_rows(X, out=None, stream=None):
    """Angular similarity preprocessing: rows scaled to unit l2 norm."""
    import torch
    lib = load_library()
    N, n = X.shape
    out = torch.empty_like(X) if out is None else out
    _check(lib.fastlsh_normalize_rows(_dev_ptr(X, torch.float32, "X"), N, n, _dev_ptr(out, torch.float32, "out"),
                                      _stream_ptr(stream)), "fastlsh_normalize_rows")
    return out


def max_row_norm(X, stream=None):
    """kappa = max_r ||X[r]||_2 as a 1-element device tensor."""
    import torch
    lib = load_library()
    N, n = X.shape
    k = torch.empty((1,), dtype=torch.float32, device=X.device)
    _check(lib.fastlsh_max_row_norm(_dev_ptr(X, torch.float32, "X"), N, n, _dev_ptr(k, torch.float32, "kappa"),
                                    _stream_ptr(stream)), "fastlsh_max_row_norm")
    return k


def mips_transform(X, kappa=None, query: bool = False, stream=None):
    """MIPS transforms: P(v) = (sqrt(kappa^2 - ||v||^2), v) for data,
    Q(u) = (0, u) for queries; returns f32 [N, n+1]."""
    import torch
    lib = load_library()
    N, n = X.shape
    out = torch.empty((N, n + 1), dtype=torch.float32, device=X.device)
    kp = _dev_ptr(kappa, torch.float32, "kappa") if kappa is not None else ctypes.c_void_p(0)
    _check(lib.fastlsh_mips_transform(_dev_ptr(X, torch.float32, "X"), N, n, kp, 1 if query else 0,
                                      _dev_ptr(out, torch.float32, "out"), _stream_ptr(stream)),
           "fastlsh_mips_transform")
    return out


def hash_keys(params: Params, keys: Keys | None, X, codes=None, keys_out=None, stream=None,
              with_codes: bool = True, col0: int = 0):
    """One step of the hot path: codes (Eq. 5) then compound keys, on the same stream.

    with_codes=False (params packed with set_table_size(K)): keys only, built in the hashing
    kernel's epilogue; codes are never written. keys_out may be a wider [L, ldk] table with the
    N keys of each table written to columns [col0, col0 + N)."""
    import torch
    params._ready()
    _check_X(params, X)
    N = X.shape[0]
    if with_codes and codes is None:
        codes = torch.empty((N, params.k), dtype=torch.int32, device=X.device)
    if codes is not None:
        _check_out(codes, N, params.k, "codes")
    if keys is not None and keys.L * keys.K > params.k:
        raise ValueError(f"keys need L*K={keys.L * keys.K} <= k={params.k} codes")
    kp = ctypes.c_void_p(0)
    ldk = N
    if keys is not None:
        if keys_out is None:
            keys_out = torch.empty((keys.L, N + col0), dtype=torch.int64, device=X.device)
        ldk = keys_out.shape[1]
        if keys_out.shape[0] != keys.L or col0 < 0 or col0 + N > ldk:
            raise ValueError("keys_out must be [L, ldk] with col0 + N <= ldk")
        kp = ctypes.c_void_p(_dev_ptr(keys_out, torch.int64, "keys").value + 8 * col0)
    cp = _dev_ptr(codes, torch.int32, "codes") if codes is not None else ctypes.c_void_p(0)
    _check(params._lib.fastlsh_hash_keys(params._h, keys._h if keys is not None else None,
                                         _dev_ptr(X, torch.float32, "X"), N, cp, kp, ldk, _stream_ptr(stream)),
           "fastlsh_hash_keys")
    return codes, keys_out


def hash_keys_multicast(params: Params, keys: Keys, X, mc_ptr: int, ldk: int, col0: int = 0, codes=None,
                        with_codes: bool = True, stream=None):
    """Hash + keys with the key all-gather fused in (fastlsh_hash_keys_multicast): the keys of X's rows
    are written with multimem.st to columns [col0, col0 + N) of the [L, ldk] u64 table whose multicast
    address is mc_ptr (torch symmetric memory), i.e. into every GPU's copy of the table. K1j only."""
    import torch
    params._ready()
    _check_X(params, X)
    N = X.shape[0]
    if keys.L * keys.K > params.k:
        raise ValueError(f"keys need L*K={keys.L * keys.K} <= k={params.k} codes")
    if col0 < 0 or col0 + N > ldk or not mc_ptr:
        raise ValueError("need a multicast pointer and col0 + N <= ldk")
    if with_codes and codes is None:
        codes = torch.empty((N, params.k), dtype=torch.int32, device=X.device)
    if codes is not None:
        _check_out(codes, N, params.k, "codes")
    cp = _dev_ptr(codes, torch.int32, "codes") if codes is not None else ctypes.c_void_p(0)
    _check(params._lib.fastlsh_hash_keys_multicast(params._h, keys._h, _dev_ptr(X, torch.float32, "X"), N, cp,
                                                   ctypes.c_void_p(int(mc_ptr) + 8 * col0), ldk, _stream_ptr(stream)),
           "fastlsh_hash_keys_multicast")
    return codes


def hash_host(params: Params, keys: Keys | None, X_host, codes_host=None, keys_host=None,
              chunk_rows: int = 65536, with_codes: bool = True):
    """End-to-end entry point on HOST buffers (numpy or pinned torch CPU tensors). with_codes=False
    (keys required): only the keys come back to the host."""
    import torch
    params._ready()
    if isinstance(X_host, np.ndarray):
        X_host = torch.from_numpy(np.ascontiguousarray(X_host, dtype=np.float32))
    if X_host.is_cuda or X_host.dtype != torch.float32 or not X_host.is_contiguous():
        raise TypeError("X_host must be a contiguous float32 host tensor")
    _check_X(params, X_host, "X_host")
    N = X_host.shape[0]
    if not with_codes and keys is None:
        raise ValueError("with_codes=False needs keys")
    if codes_host is None and with_codes:
        codes_host = torch.empty((N, params.k), dtype=torch.int32, pin_memory=X_host.is_pinned())
    if codes_host is not None:
        if codes_host.is_cuda or codes_host.dtype != torch.int32 or not codes_host.is_contiguous():
            raise TypeError("codes_host must be a contiguous int32 host tensor")
        _check_out(codes_host, N, params.k, "codes_host")
    kp = ctypes.c_void_p(0)
    if keys is not None:
        if keys.L * keys.K > params.k:
            raise ValueError(f"keys need L*K={keys.L * keys.K} <= k={params.k} codes")
        if keys_host is None:
            keys_host = torch.empty((keys.L, N), dtype=torch.int64, pin_memory=X_host.is_pinned())
        if keys_host.is_cuda or keys_host.dtype != torch.int64 or not keys_host.is_contiguous():
            raise TypeError("keys_host must be a contiguous int64 host tensor")
        _check_out(keys_host, keys.L, N, "keys_host")
        kp = ctypes.c_void_p(keys_host.data_ptr())
    _check(params._lib.fastlsh_hash_host(params._h, keys._h if keys is not None else None,
                                         ctypes.c_void_p(X_host.data_ptr()), N,
                                         ctypes.c_void_p(codes_host.data_ptr() if codes_host is not None else 0), kp,
                                         chunk_rows),
           "fastlsh_hash_host")
    return codes_host, keys_host


def read_flags(params: Params, reset: bool = False, stream=None):
    params._ready()
    nf, sat = ctypes.c_uint64(), ctypes.c_uint64()
    _check(params._lib.fastlsh_read_flags(params._h, ctypes.byref(nf), ctypes.byref(sat), int(reset),
                                          _stream_ptr(stream)), "fastlsh_read_flags")
    return nf.value, sat.value


def bandwidth_probe(inp, out, rows: int, read_bytes: int, write_bytes: int, stream=None):
    """Diagnostic streaming kernel (fastlsh_bandwidth_probe): `rows` rows of read_bytes read from
    `inp` and write_bytes written to `out` (CUDA tensors of at least rows * bytes)."""
    lib = load_library()
    if inp.numel() * inp.element_size() < rows * read_bytes or out.numel() * out.element_size() < rows * write_bytes:
        raise ValueError("probe buffers too small")
    _check(lib.fastlsh_bandwidth_probe(ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()), rows,
                                       read_bytes, write_bytes, _stream_ptr(stream)), "fastlsh_bandwidth_probe")


class MulticastTable:
    """An [L, ldk] int64 table on the current GPU mapped both normally (`table`, a torch view) and
    through an NVSwitch multicast object (`mc_ptr`, for fastlsh_hash_keys_multicast):
    fastlsh_multicast_alloc. Raises FastLSHError(EUNSUPPORTED) where multicast is unavailable."""

    def __init__(self, L: int, ldk: int):
        import torch
        lib = load_library()
        self._lib = lib
        uc, mc, h = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib.fastlsh_multicast_alloc(L * ldk * 8, ctypes.byref(uc), ctypes.byref(mc), ctypes.byref(h)),
               "fastlsh_multicast_alloc")
        self._h = h
        self.mc_ptr = mc.value

        class _Arr:  # zero-copy torch view of the unicast mapping
            __cuda_array_interface__ = {"shape": (L, ldk), "typestr": "<i8", "data": (uc.value, False),
                                        "version": 3, "strides": None}
        self.table = torch.as_tensor(_Arr(), device="cuda")

    def close(self):
        if self._h is not None and self._h.value:
            self.table = None
            self._lib.fastlsh_multicast_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
