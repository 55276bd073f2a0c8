"""Thin Python binding of libmaple.so (include/maple.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module converts numpy / torch buffers
to pointers and back, and raises MapleError on a nonzero status. There is no CPU fallback: if the shared
library (or a CUDA device) is missing, load() raises.

Low-level functions keep the C names (maple_create, maple_extract, ...); `Context` / `DirSet` wrap them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmaple.so")
_lib = None

ERRORS = {
    -1: "BAD_ARG", -2: "BAD_BOUNDS", -3: "RANK_DEFICIENT", -4: "FULL_RANK", -5: "OVERFLOW", -6: "RANGE",
    -7: "CUDA", -8: "OOM", -9: "CAPACITY", -10: "INFEASIBLE", -11: "COMM",
}
OBJ_QUADRATIC, OBJ_SEPARABLE, OBJ_TABLE = 0, 1, 2
STATUS_OK, STATUS_NO_FEASIBLE = 0, 1

class maple_objective(C.Structure):
    _fields_ = [("kind", C.c_int32), ("Q", C.POINTER(C.c_double)), ("c", C.POINTER(C.c_double)), ("c0", C.c_double)]


# (name, restype, argtypes) for every exported symbol of include/maple.h
_P = C.c_void_p
_SIGS = [
    ("maple_create", C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, C.c_int, C.POINTER(_P)]),
    ("maple_destroy", None, [_P]),
    ("maple_kernel_basis", C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    ("maple_set_stream", C.c_int, [_P, _P]),
    ("maple_set_extract_params", C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32]),
    ("maple_get_basis", C.c_int, [_P, _P]),
    ("maple_get_pinv", C.c_int, [_P, _P]),
    ("maple_dim_n", C.c_int32, [_P]),
    ("maple_dim_d", C.c_int32, [_P]),
    ("maple_last_error", C.c_char_p, [_P]),
    ("maple_extract", C.c_int, [_P, C.c_int64, C.c_int32, C.c_double, C.c_uint64, C.POINTER(_P)]),
    ("maple_extract_range", C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_double, C.c_uint64,
                                      C.POINTER(_P)]),
    ("maple_dirset_merge", C.c_int, [_P, _P, C.c_int64, C.c_int32, C.POINTER(_P)]),
    ("maple_dirset_size", C.c_int64, [_P]),
    ("maple_dirset_pool_size", C.c_int64, [_P]),
    ("maple_dirset_copy", C.c_int, [_P, _P]),
    ("maple_dirset_device_rows", _P, [_P]),
    ("maple_dirset_stride", C.c_int32, [_P]),
    ("maple_dirset_copy_i8", C.c_int, [_P, _P]),
    ("maple_dirset_copy_raw", C.c_int, [_P, _P]),
    ("maple_dirset_copy_device", C.c_int, [_P, _P]),
    ("maple_dirset_free", None, [_P]),
    ("maple_dirset_from_host", C.c_int, [_P, _P, C.c_int64, C.c_int32, C.POINTER(_P)]),
    ("maple_set_filter_minimal", C.c_int, [_P, C.c_int32]),
    ("maple_dirset_keep_range", C.c_int, [_P, _P, C.c_int64, C.c_int64, _P]),
    ("maple_dirset_select", C.c_int, [_P, _P, _P, C.POINTER(_P)]),
    ("maple_augment", C.c_int, [_P, _P, C.POINTER(maple_objective), _P, _P, C.c_int32, _P, _P, _P, _P]),
    ("maple_augment_many", C.c_int, [_P, _P, C.c_int32, C.POINTER(maple_objective), _P, _P, C.c_int32, _P, _P]),
    ("maple_debug_descent", C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_double, C.c_uint64, _P, _P]),
    ("maple_set_debug", C.c_int, [_P, C.c_int32]),
    ("maple_debug_trace", C.c_int, [_P, C.c_int32, _P]),
    ("maple_debug_candidates", C.c_int64, [_P, _P, C.c_int64]),
    ("maple_last_timings", C.c_int, [_P, _P, _P]),
    ("maple_kernel_launches", C.c_int64, [_P]),
    ("maple_set_descent_kernel", C.c_int, [_P, C.c_int32]),
    ("maple_descent_kernel", C.c_int, [_P]),
    ("maple_set_filter_algorithm", C.c_int, [_P, C.c_int32]),
    ("maple_set_descent_variant", C.c_int, [_P, C.c_int32, C.c_int32]),
    ("maple_selftest_umma", C.c_int, [C.c_int, _P, _P, _P, _P, _P, _P]),
    ("maple_selftest_pair", C.c_int, [C.c_int, _P, _P, _P, _P, _P, _P]),
    ("maple_feasible_starts", C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, _P,
                                        C.c_int32, _P, _P]),
]


class MapleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"MAPLE_ERR_{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.name = ERRORS.get(code, str(code))


def load(path: str = LIB_PATH):
    """Load libmaple.so (no fallback: raises if it is missing or lacks a symbol)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run __graft_entry__.build() (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return [s[0] for s in _SIGS]


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc, ctx=None):
    if rc != 0:
        msg = _lib.maple_last_error(ctx).decode() if ctx else ""
        raise MapleError(rc, msg)


def maple_kernel_basis(A):
    """Host-only lattice step of maple_create: returns (B, B+) as computed by the library."""
    load()
    A = np.ascontiguousarray(A, dtype=np.int32)
    m, n = A.shape
    B = np.zeros((n, n - m), np.int32)
    Bp = np.zeros((n - m, n), np.float64)
    rc = _lib.maple_kernel_basis(_ptr(A), m, n, _ptr(B), _ptr(Bp))
    if rc != 0:
        raise MapleError(rc, "maple_kernel_basis")
    return B, Bp


def maple_selftest_umma(A1, B1, A2, B2, device=0):
    """Single-tile tcgen05 products D1 = A1 B1^T (tf32) and D2 = A2 B2^T (f16) computed on the device."""
    load()
    A1, B1, A2, B2 = (np.ascontiguousarray(x, dtype=np.float32) for x in (A1, B1, A2, B2))
    D1 = np.zeros((128, 64), np.float32)
    D2 = np.zeros((128, 48), np.float32)
    rc = _lib.maple_selftest_umma(device, _ptr(A1), _ptr(B1), _ptr(D1), _ptr(A2), _ptr(B2), _ptr(D2))
    if rc != 0:
        raise MapleError(rc, "maple_selftest_umma")
    return D1, D2


def maple_selftest_pair(Ah, Bh, A8, B8, device=0):
    """CTA-pair tcgen05 products (f16 and i8, TMA-loaded B split across the pair): raw TMEM read-backs
    raw1 (2, 128, 80) fp32 and raw2 (2, 128, 64) int32 of each CTA (lanes x columns)."""
    load()
    Ah = np.ascontiguousarray(Ah, dtype=np.float16).view(np.uint16)
    Bh = np.ascontiguousarray(Bh, dtype=np.float16).view(np.uint16)
    A8, B8 = (np.ascontiguousarray(x, dtype=np.int8) for x in (A8, B8))
    raw1 = np.zeros((2, 128, 80), np.float32)
    raw2 = np.zeros((2, 128, 64), np.int32)
    rc = _lib.maple_selftest_pair(device, _ptr(Ah), _ptr(Bh), _ptr(A8), _ptr(B8), _ptr(raw1), _ptr(raw2))
    if rc != 0:
        raise MapleError(rc, "maple_selftest_pair")
    return raw1, raw2


class DirSet:
    """A device-resident direction set (canonical rows, lexicographically sorted)."""

    def __init__(self, ctx: "Context", handle):
        self.ctx = ctx
        self.h = handle

    @property
    def size(self) -> int:
        return int(_lib.maple_dirset_size(self.h))

    @property
    def pool_size(self) -> int:
        return int(_lib.maple_dirset_pool_size(self.h))

    @property
    def stride(self) -> int:
        return int(_lib.maple_dirset_stride(self.h))

    @property
    def device_ptr(self) -> int:
        return _lib.maple_dirset_device_rows(self.h) or 0

    def rows(self, dtype=np.int32) -> np.ndarray:
        """Host copy of the rows, (size, n); dtype int32 (default) or int8 (one strided copy, 4x fewer bytes)."""
        if np.dtype(dtype) == np.int8:
            out = np.empty((self.size, self.ctx.n), dtype=np.int8)
            _check(_lib.maple_dirset_copy_i8(self.h, _ptr(out) if out.size else None), self.ctx.h)
            return out
        out = np.zeros((self.size, self.ctx.n), dtype=np.int32)
        _check(_lib.maple_dirset_copy(self.h, _ptr(out) if out.size else None), self.ctx.h)
        return out

    def rows_pinned(self) -> np.ndarray:
        """Host rows (size, n) int8 from ONE contiguous DMA into page-locked memory (the stored size x stride rows;
        a strided view drops the zero padding). The pinned buffer is allocated by torch when it is available."""
        k, st = self.size, self.stride
        try:
            import torch
            buf = torch.empty((max(k, 1), st), dtype=torch.int8, pin_memory=True).numpy()
        except Exception:
            buf = np.empty((max(k, 1), st), dtype=np.int8)
        if k:
            _check(_lib.maple_dirset_copy_raw(self.h, _ptr(buf)), self.ctx.h)
        return buf[:k, :self.ctx.n]

    def copy_device(self, dst_ptr: int):
        """Copy the rows (size x stride int8) into device memory at dst_ptr."""
        _check(_lib.maple_dirset_copy_device(self.h, C.c_void_p(dst_ptr)), self.ctx.h)

    def free(self):
        if self.h:
            _lib.maple_dirset_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """maple_create(A, l, u): host-exact HNF + LLL + B+ and device upload."""

    def __init__(self, A, l, u, device: int = 0):
        load()
        A = np.ascontiguousarray(A, dtype=np.int32)
        l = np.ascontiguousarray(l, dtype=np.int32)
        u = np.ascontiguousarray(u, dtype=np.int32)
        self.m, self.n = A.shape
        h = C.c_void_p()
        rc = _lib.maple_create(_ptr(A), self.m, self.n, _ptr(l), _ptr(u), device, C.byref(h))
        if rc != 0:
            raise MapleError(rc, "maple_create")
        self.h = h
        self.d = int(_lib.maple_dim_d(h))
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            _lib.maple_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- configuration ----
    def set_stream(self, stream_handle: int):
        _check(_lib.maple_set_stream(self.h, C.c_void_p(stream_handle)), self.h)

    def set_params(self, lambda1=0.85, lambda2=1.0, beta1=0.9, beta2=0.999, eps=1e-8, filter_minimal=True):
        _check(_lib.maple_set_extract_params(self.h, lambda1, lambda2, beta1, beta2, eps, int(filter_minimal)), self.h)

    def set_descent_kernel(self, which: int):
        _check(_lib.maple_set_descent_kernel(self.h, which), self.h)

    def set_descent_variant(self, optimizer: str = "adam", harvest_final: bool = False):
        """Alg. 3 line 8 update ('adam', 'gd', 'signgd') and final-only harvest (maple_set_descent_variant)."""
        code = {"adam": 0, "gd": 1, "signgd": 2}[optimizer]
        _check(_lib.maple_set_descent_variant(self.h, code, int(harvest_final)), self.h)

    def set_filter_algorithm(self, which: int):
        """0 auto, 1 tiled, 2 indexed, 3 level-synchronous (maple_set_filter_algorithm): same kept set, different
        pair enumeration."""
        _check(_lib.maple_set_filter_algorithm(self.h, which), self.h)

    @property
    def descent_kernel(self) -> str:
        """'simt', 'tc' or 'tcp' (CTA-pair tcgen05, large shapes): the descent kernel the next extraction
        launches."""
        r = _lib.maple_descent_kernel(self.h)
        _check(min(r, 0), self.h)
        return {1: "simt", 2: "tc", 4: "tcp"}[r]

    def debug_trace(self, enable: bool = True):
        """Arm (enable) or read back the CTA-pair kernel's per-step timeline: (2, 16, 16) uint64 ns stamps."""
        out = np.zeros((2, 16, 16), np.uint64)
        _check(_lib.maple_debug_trace(self.h, 1 if enable else 0, _ptr(out)), self.h)
        return out

    def set_debug(self, keep_candidates: bool):
        _check(_lib.maple_set_debug(self.h, int(keep_candidates)), self.h)

    @property
    def B(self) -> np.ndarray:
        out = np.zeros((self.n, self.d), dtype=np.int32)
        _check(_lib.maple_get_basis(self.h, _ptr(out)), self.h)
        return out

    @property
    def Bp(self) -> np.ndarray:
        out = np.zeros((self.d, self.n), dtype=np.float64)
        _check(_lib.maple_get_pinv(self.h, _ptr(out)), self.h)
        return out

    # ---- extraction ----
    def extract(self, n_starts, steps, step_size, seed) -> DirSet:
        h = C.c_void_p()
        _check(_lib.maple_extract(self.h, int(n_starts), int(steps), float(step_size), int(seed), C.byref(h)), self.h)
        return DirSet(self, h)

    def extract_range(self, n_starts, begin, end, steps, step_size, seed) -> DirSet:
        h = C.c_void_p()
        _check(_lib.maple_extract_range(self.h, int(n_starts), int(begin), int(end), int(steps), float(step_size),
                                        int(seed), C.byref(h)), self.h)
        return DirSet(self, h)

    def merge_device(self, ptr: int, k: int, stride: int) -> DirSet:
        h = C.c_void_p()
        _check(_lib.maple_dirset_merge(self.h, C.c_void_p(ptr), int(k), int(stride), C.byref(h)), self.h)
        return DirSet(self, h)

    def set_filter_minimal(self, on: bool):
        """maple_set_filter_minimal: whether extract / merge apply the ⊑-minimality filter (default on)."""
        _check(_lib.maple_set_filter_minimal(self.h, int(bool(on))), self.h)

    def keep_range(self, pool: DirSet, begin: int, end: int, keep_ptr: int):
        """maple_dirset_keep_range: keep bytes of pool rows [begin, end) into the device buffer at keep_ptr."""
        _check(_lib.maple_dirset_keep_range(self.h, pool.h, int(begin), int(end), C.c_void_p(keep_ptr)), self.h)

    def select(self, pool: DirSet, keep_ptr: int) -> DirSet:
        """maple_dirset_select: the pool rows whose keep byte (device buffer, pool.size bytes) is nonzero."""
        h = C.c_void_p()
        _check(_lib.maple_dirset_select(self.h, pool.h, C.c_void_p(keep_ptr), C.byref(h)), self.h)
        return DirSet(self, h)

    def dirset_from_host(self, rows, filter_minimal=True) -> DirSet:
        rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int32).reshape(-1, self.n))
        h = C.c_void_p()
        _check(_lib.maple_dirset_from_host(self.h, _ptr(rows) if rows.size else None, rows.shape[0],
                                           int(filter_minimal), C.byref(h)), self.h)
        return DirSet(self, h)

    def debug_descent(self, n_starts, begin, end, steps, step_size, seed):
        Z = np.zeros((end - begin, self.d), dtype=np.float32)
        Z0 = np.zeros((end - begin, self.d), dtype=np.float64)
        _check(_lib.maple_debug_descent(self.h, int(n_starts), int(begin), int(end), int(steps), float(step_size),
                                        int(seed), _ptr(Z), _ptr(Z0)), self.h)
        return Z, Z0

    def candidates(self) -> np.ndarray:
        k = int(_lib.maple_debug_candidates(self.h, None, 0))
        out = np.zeros((k, self.n), dtype=np.int32)
        if k:
            _lib.maple_debug_candidates(self.h, _ptr(out), k)
        return out

    def timings(self):
        e = np.zeros(6, np.float32)
        a = np.zeros(3, np.float32)
        _check(_lib.maple_last_timings(self.h, _ptr(e), _ptr(a)), self.h)
        return {"descent": float(e[0]), "dedupe": float(e[1]), "check": float(e[2]), "filter": float(e[3]),
                "sort": float(e[4]), "extract_total": float(e[5]), "aug_precompute": float(a[0]),
                "aug_iterate": float(a[1]), "augment_total": float(a[2])}

    def launches(self) -> int:
        return int(_lib.maple_kernel_launches(self.h))

    # ---- Eq. 4 feasible starts ----
    def feasible_starts(self, b, k, steps, step_size, lambda3=0.1, seed=0, debug=False):
        """maple_feasible_starts: (sorted distinct feasible points (count x n), final iterates or None)."""
        b = np.ascontiguousarray(b, dtype=np.int32)
        out = np.zeros((k, self.n), np.int32)
        cnt = np.zeros(1, np.int32)
        X = np.zeros((k, self.n), np.float32) if debug else None
        _check(_lib.maple_feasible_starts(self.h, _ptr(b), int(k), int(steps), float(step_size), float(lambda3),
                                          int(seed), _ptr(out), k, _ptr(cnt), _ptr(X) if debug else None), self.h)
        return out[:min(int(cnt[0]), k)], X

    # ---- augmentation ----
    @staticmethod
    def _objective(Q, c, c0, kind):
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        c = np.ascontiguousarray(np.zeros(1) if c is None else c, dtype=np.float64)   # OBJ_TABLE: c unused
        ob = maple_objective(kind, Q.ctypes.data_as(C.POINTER(C.c_double)), c.ctypes.data_as(C.POINTER(C.c_double)),
                             float(c0))
        return ob, (Q, c)

    def augment(self, ds: DirSet, Q, c, c0, b, x0, kind=OBJ_QUADRATIC):
        """maple_augment: returns (x_best, f_best, status, iters per incumbent)."""
        ob, keep = self._objective(Q, c, c0, kind)
        b = np.ascontiguousarray(b, dtype=np.int32)
        x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.int32).reshape(-1, self.n))
        k0 = x0.shape[0]
        xb = np.zeros(self.n, np.int32)
        fb = np.zeros(1, np.float64)
        st = np.zeros(1, np.int32)
        it = np.zeros(max(k0, 1), np.int32)
        _check(_lib.maple_augment(self.h, ds.h, C.byref(ob), _ptr(b), _ptr(x0) if k0 else None, k0, _ptr(xb), _ptr(fb),
                                  _ptr(st), _ptr(it)), self.h)
        del keep
        return xb, float(fb[0]), int(st[0]), it[:k0]

    def augment_many(self, ds: DirSet, Qs, cs, c0s, bs, X0s, kind=OBJ_QUADRATIC):
        """maple_augment_many over n_inst instances sharing A and the direction set (configs[3]). kind: one
        objective kind for all instances, or one per instance (TABLE cannot be mixed with the quadratic kinds)."""
        n_inst = len(Qs)
        obs = (maple_objective * n_inst)()
        keep = []
        for t in range(n_inst):
            ob, k = self._objective(Qs[t], None if cs is None else cs[t], c0s[t],
                                   kind[t] if isinstance(kind, (list, tuple)) else kind)
            obs[t] = ob
            keep.append(k)
        b = np.ascontiguousarray(np.asarray(bs, dtype=np.int32).reshape(n_inst, self.m))
        X0 = np.ascontiguousarray(np.asarray(X0s, dtype=np.int32).reshape(n_inst, -1, self.n))
        k0 = X0.shape[1]
        xb = np.zeros((n_inst, self.n), np.int32)
        fb = np.zeros(n_inst, np.float64)
        _check(_lib.maple_augment_many(self.h, ds.h, n_inst, obs, _ptr(b), _ptr(X0), k0, _ptr(xb), _ptr(fb)), self.h)
        del keep
        return xb, fb
