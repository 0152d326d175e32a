"""Thin ctypes binding of libnsrgs.so (include/nsrgs.h).

Argument marshalling only: every step of the NS-RGS path runs in the library's CUDA
kernels.  PyTorch is used for the CUDA stream handle and (optionally) device tensors;
host arrays are NumPy.  There is no CPU fallback: if libnsrgs.so is missing, importing
this module raises.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnsrgs.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libnsrgs.so not built ({_LIB_PATH}); run `python -m paper_2604_07372_b200.build` "
                      "or __graft_entry__.build() — there is no CPU fallback")
_lib = ct.CDLL(_LIB_PATH)

F32, F64 = 0, 1
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "STATE", 3: "CUDA", 4: "NCCL", 5: "OOM", 6: "DIVERGENCE",
          7: "SINGULAR", 8: "EIG_NOT_CONVERGED", 9: "NONFINITE"}


class NSRGSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"nsrgs {STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Desc(ct.Structure):
    _fields_ = [("n", ct.c_int64), ("d", ct.c_int32), ("dtype", ct.c_int32), ("rank", ct.c_int32),
                ("world", ct.c_int32), ("device", ct.c_int32), ("nccl_unique_id", ct.c_void_p),
                ("cuda_stream", ct.c_void_p)]


class Plan(ct.Structure):
    _fields_ = [(k, ct.c_int64) for k in ("n_local", "node0", "rows_local", "row0", "col_tile",
                                          "tiles_per_rank", "x_elems", "x_slice_elems")]


class Stats(ct.Structure):
    _fields_ = [("grid", ct.c_int32), ("threads", ct.c_int32), ("stages", ct.c_int32),
                ("rows_per_panel", ct.c_int32), ("cut_panels", ct.c_int32), ("panels", ct.c_int64),
                ("smem_bytes", ct.c_int64), ("panel_ms_total", ct.c_double), ("panel_launches", ct.c_int64),
                ("kernel_launches", ct.c_int64), ("ns_region_max", ct.c_double), ("a_fro2", ct.c_double),
                ("symmetric", ct.c_int32), ("a_bytes_per_pass", ct.c_int64), ("p2p", ct.c_int32),
                ("bsr", ct.c_int32), ("bsr_nnzb", ct.c_int64), ("bsr_slab", ct.c_int32), ("bsr_g4", ct.c_int32),
                ("wide_tc", ct.c_int32)]


_P = ct.c_void_p
_SIGS = {
    "nsrgs_version": ([], ct.c_int),
    "nsrgs_plan": ([ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int32, ct.POINTER(Plan)], ct.c_int),
    "nsrgs_pack_host": ([ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int32, _P, _P], ct.c_int),
    "nsrgs_unpack_host": ([ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int32, _P, _P], ct.c_int),
    "nsrgs_get_nccl_unique_id": ([_P], ct.c_int),
    "nsrgs_create": ([ct.POINTER(Desc), ct.POINTER(_P)], ct.c_int),
    "nsrgs_destroy": ([_P], ct.c_int),
    "nsrgs_last_error": ([_P], ct.c_char_p),
    "nsrgs_attach_A": ([_P, _P, ct.c_int64], ct.c_int),
    "nsrgs_generate": ([_P, ct.c_uint64, ct.c_double, _P], ct.c_int),
    "nsrgs_generate_observed": ([_P, ct.c_uint64, ct.c_double, ct.c_double, _P], ct.c_int),
    "nsrgs_copy_A_rows": ([_P, ct.c_int64, ct.c_int64, _P], ct.c_int),
    "nsrgs_generate_observed_bsr": ([_P, ct.c_uint64, ct.c_double, ct.c_double, _P], ct.c_int),
    "nsrgs_attach_A_bsr": ([_P, _P, _P, _P, ct.c_int64], ct.c_int),
    "nsrgs_get_A_bsr": ([_P, ct.POINTER(ct.c_int64), _P, _P, _P], ct.c_int),
    "nsrgs_init_spectral": ([_P, ct.c_uint64, ct.c_int, ct.c_double, ct.POINTER(ct.c_int)], ct.c_int),
    "nsrgs_step": ([_P, ct.c_double, ct.c_int, ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_run": ([_P, ct.c_int, ct.c_double, ct.c_int, ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_objective": ([_P, ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_objective_fp64": ([_P, ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_gpm_run": ([_P, ct.c_int, ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_solve": ([_P, ct.c_int, ct.c_int, ct.c_double, ct.c_int, ct.c_double, ct.POINTER(ct.c_int),
                     ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_alignment_error": ([_P, _P, ct.c_int, ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_set_X": ([_P, _P, ct.c_int], ct.c_int),
    "nsrgs_get_X": ([_P, _P, ct.c_int], ct.c_int),
    "nsrgs_get_stats": ([_P, ct.POINTER(Stats)], ct.c_int),
    "nsrgs_set_symmetric": ([_P, ct.c_int], ct.c_int),
    "nsrgs_debug_timestamps": ([_P, ct.c_int, _P], ct.c_int),
    "nsrgs_debug_link_peers": ([_P, ct.c_int], ct.c_int),
    "nsrgs_debug_group": ([_P, ct.c_int], ct.c_int),
    "nsrgs_probe_read_stream": ([_P, ct.c_int64, _P, ct.c_int, ct.POINTER(ct.c_double)], ct.c_int),
    "nsrgs_reset_stats": ([_P, ct.c_int], ct.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def _np_dtype(dtype: int):
    return np.float32 if dtype == F32 else np.float64


def version() -> int:
    return _lib.nsrgs_version()


def link_peers(solvers) -> None:
    """Test-only (NSRGS_EMULATE_RANKS=1): fused P2P exchange between rank contexts of one process."""
    arr = (_P * len(solvers))(*[s._h.value for s in solvers])
    rc = _lib.nsrgs_debug_link_peers(arr, len(solvers))
    if rc != 0:
        raise NSRGSError(rc, (_lib.nsrgs_last_error(solvers[0]._h) or b"").decode())


def link_group(solvers) -> None:
    """Test-only (NSRGS_EMULATE_RANKS=1): in-process rank group with real collectives; drive
    each rank's calls from its own thread (see nsrgs_debug_group)."""
    arr = (_P * len(solvers))(*[s._h.value for s in solvers])
    rc = _lib.nsrgs_debug_group(arr, len(solvers))
    if rc != 0:
        raise NSRGSError(rc, (_lib.nsrgs_last_error(solvers[0]._h) or b"").decode())


def probe_read_stream(buf, stream, reps: int = 5) -> float:
    """HBM read-stream ceiling (GB/s) over the device tensor `buf` (nsrgs_probe_read_stream)."""
    g = ct.c_double(0.0)
    rc = _lib.nsrgs_probe_read_stream(buf.data_ptr(), buf.numel() * buf.element_size(), _P(stream.cuda_stream), reps,
                                      ct.byref(g))
    if rc != 0:
        raise NSRGSError(rc, "probe_read_stream")
    return g.value


def plan(n: int, d: int, world: int = 1, rank: int = 0) -> dict:
    p = Plan()
    s = _lib.nsrgs_plan(n, d, world, rank, ct.byref(p))
    if s:
        raise NSRGSError(s, "unsupported (n, d, world, rank)")
    return {k: getattr(p, k) for k, _ in Plan._fields_}


def pack_host(stack: np.ndarray, n: int, d: int, world: int) -> np.ndarray:
    """nd x d stack -> device tile layout (host arrays; see nsrgs_plan)."""
    dt = F32 if stack.dtype == np.float32 else F64
    stack = np.ascontiguousarray(stack)
    out = np.empty(plan(n, d, world)["x_elems"], dtype=stack.dtype)
    s = _lib.nsrgs_pack_host(n, d, world, dt, stack.ctypes.data, out.ctypes.data)
    if s:
        raise NSRGSError(s, "pack_host")
    return out


def unpack_host(tiled: np.ndarray, n: int, d: int, world: int) -> np.ndarray:
    dt = F32 if tiled.dtype == np.float32 else F64
    tiled = np.ascontiguousarray(tiled)
    out = np.empty((n * d, d), dtype=tiled.dtype)
    s = _lib.nsrgs_unpack_host(n, d, world, dt, tiled.ctypes.data, out.ctypes.data)
    if s:
        raise NSRGSError(s, "unpack_host")
    return out


def get_nccl_unique_id() -> bytes:
    buf = ct.create_string_buffer(128)
    s = _lib.nsrgs_get_nccl_unique_id(buf)
    if s:
        raise NSRGSError(s, "ncclGetUniqueId")
    return buf.raw


class Solver:
    """One NS-RGS context (one per process / GPU).  Methods mirror the C-ABI names."""

    def __init__(self, n: int, d: int, dtype: int = F32, rank: int = 0, world: int = 1, device: int = 0,
                 nccl_id: bytes | None = None, stream=None):
        import torch  # CUDA stream handle only

        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.n, self.d, self.dtype, self.rank, self.world, self.device = n, d, dtype, rank, world, device
        self.np_dtype = _np_dtype(dtype)
        self._stream = stream
        self._id = ct.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        desc = Desc(n, d, dtype, rank, world, device, ct.cast(self._id, _P) if self._id is not None else None,
                    _P(stream.cuda_stream))
        h = _P()
        s = _lib.nsrgs_create(ct.byref(desc), ct.byref(h))
        if s:
            raise NSRGSError(s, _lib.nsrgs_last_error(None).decode())
        self._h = h

    # ------------------------------------------------------------------ plumbing
    def _check(self, s: int):
        if s:
            raise NSRGSError(s, _lib.nsrgs_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            _lib.nsrgs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @staticmethod
    def _ptr(x):
        """(pointer, on_device) of a NumPy array or torch tensor (contiguous)."""
        if isinstance(x, np.ndarray):
            assert x.flags["C_CONTIGUOUS"]
            return x.ctypes.data, 0
        assert x.is_contiguous()
        return x.data_ptr(), int(x.is_cuda)

    # ------------------------------------------------------------------ C-ABI calls
    def generate(self, seed: int, sigma: float, want_Z: bool = True, p: float = 1.0, storage: str = "dense"):
        """storage="dense" (row-major shard) or "bsr" (observed blocks only)."""
        Z = np.empty((self.n, self.d, self.d), dtype=self.np_dtype) if want_Z else None
        zp = Z.ctypes.data if want_Z else None
        if storage == "bsr":
            self._check(_lib.nsrgs_generate_observed_bsr(self._h, seed, sigma, p, zp))
        elif storage != "dense":
            raise ValueError(storage)
        elif p == 1.0:
            self._check(_lib.nsrgs_generate(self._h, seed, sigma, zp))
        else:
            self._check(_lib.nsrgs_generate_observed(self._h, seed, sigma, p, zp))
        return Z

    def attach_A(self, A_shard, lda: int | None = None):
        ptr, dev = self._ptr(A_shard)
        assert dev, "attach_A needs a device tensor"
        self._A_ref = A_shard
        self._check(_lib.nsrgs_attach_A(self._h, ptr, lda if lda is not None else A_shard.stride(0)))

    def attach_A_bsr(self, rowptr, col, vals):
        """Borrow a caller-owned block-sparse A (device tensors: int64 rowptr, int32 col, float32 vals)."""
        for t in (rowptr, col, vals):
            assert t.is_cuda and t.is_contiguous()
        self._A_ref = (rowptr, col, vals)
        nnzb = col.numel()
        self._check(_lib.nsrgs_attach_A_bsr(self._h, rowptr.data_ptr(), col.data_ptr(), vals.data_ptr(), nnzb))

    def get_A_bsr(self):
        """(rowptr int64[n_local+1], col int32[nnzb], vals float32[nnzb, d, d]) on the host."""
        nnzb = ct.c_int64(0)
        self._check(_lib.nsrgs_get_A_bsr(self._h, ct.byref(nnzb), None, None, None))
        nl = self.n // self.world
        rowptr = np.empty(nl + 1, dtype=np.int64)
        col = np.empty(nnzb.value, dtype=np.int32)
        vals = np.empty((nnzb.value, self.d, self.d), dtype=np.float32)
        self._check(_lib.nsrgs_get_A_bsr(self._h, ct.byref(nnzb), rowptr.ctypes.data, col.ctypes.data,
                                         vals.ctypes.data))
        return rowptr, col, vals

    def copy_A_rows(self, row0: int, nrows: int) -> np.ndarray:
        out = np.empty((nrows, self.n * self.d), dtype=self.np_dtype)
        self._check(_lib.nsrgs_copy_A_rows(self._h, row0, nrows, out.ctypes.data))
        return out

    def init_spectral(self, seed: int = 0, max_sweeps: int = 200, tol: float = 1e-5, allow_unconverged=False) -> int:
        sw = ct.c_int(0)
        s = _lib.nsrgs_init_spectral(self._h, seed, max_sweeps, tol, ct.byref(sw))
        if s == 8 and allow_unconverged:
            return sw.value
        self._check(s)
        return sw.value

    def step(self, eta: float, K: int) -> float:
        f = ct.c_double(0.0)
        self._check(_lib.nsrgs_step(self._h, eta, K, ct.byref(f)))
        return f.value

    def run(self, T: int, eta: float, K: int, trace: bool = True):
        buf = (ct.c_double * max(T, 1))() if trace else None
        self._check(_lib.nsrgs_run(self._h, T, eta, K, buf))
        return np.array(buf[:T]) if trace else None

    def gpm_run(self, T: int, trace: bool = True):
        buf = (ct.c_double * max(T, 1))() if trace else None
        self._check(_lib.nsrgs_gpm_run(self._h, T, buf))
        return np.array(buf[:T]) if trace else None

    def solve(self, algorithm: str = "ns_rgs", max_iter: int = 100, eta: float | None = None, K: int = 1,
              stop_tol: float = 1e-8):
        """Paper protocol.  Returns (iterations, F trace of length it + 1)."""
        alg = {"ns_rgs": 0, "gpm": 1}[algorithm]
        it = ct.c_int(0)
        buf = (ct.c_double * (max_iter + 1))()
        self._check(_lib.nsrgs_solve(self._h, alg, max_iter, eta if eta is not None else 1.0 / self.n, K, stop_tol,
                                     ct.byref(it), buf))
        return it.value, np.array(buf[:it.value + 1])

    def objective(self) -> float:
        f = ct.c_double(0.0)
        self._check(_lib.nsrgs_objective(self._h, ct.byref(f)))
        return f.value

    def objective_fp64(self) -> float:
        """F(X) with fp64-accumulated <X, A X> (F32 contexts; the solve stopping-rule evaluator)."""
        f = ct.c_double(0.0)
        self._check(_lib.nsrgs_objective_fp64(self._h, ct.byref(f)))
        return f.value

    def alignment_error(self, Z):
        out = (ct.c_double * 3)()
        if isinstance(Z, np.ndarray):
            Z = np.ascontiguousarray(Z, dtype=self.np_dtype)
        ptr, dev = self._ptr(Z)
        self._check(_lib.nsrgs_alignment_error(self._h, ptr, dev, out))
        return tuple(out)

    def set_X(self, X):
        if isinstance(X, np.ndarray):
            X = np.ascontiguousarray(X, dtype=self.np_dtype)
        ptr, dev = self._ptr(X)
        self._check(_lib.nsrgs_set_X(self._h, ptr, dev))

    def get_X(self, out=None) -> np.ndarray:
        if out is None:
            out = np.empty((self.n, self.d, self.d), dtype=self.np_dtype)
        ptr, dev = self._ptr(out)
        self._check(_lib.nsrgs_get_X(self._h, ptr, dev))
        return out

    def debug_timestamps(self, max_iters: int = 0):
        """Arm (max_iters > 0) or collect (0) per-CTA phase timestamps: array [iters][grid][16] ns."""
        if max_iters > 0:
            self._ts_iters = max_iters
            self._check(_lib.nsrgs_debug_timestamps(self._h, max_iters, None))
            return None
        out = np.zeros((self._ts_iters, self.stats()["grid"], 16), dtype=np.uint64)
        self._check(_lib.nsrgs_debug_timestamps(self._h, 0, out.ctypes.data))
        return out

    def set_symmetric(self, enable: bool = True):
        self._check(_lib.nsrgs_set_symmetric(self._h, int(enable)))

    def stats(self) -> dict:
        st = Stats()
        self._check(_lib.nsrgs_get_stats(self._h, ct.byref(st)))
        return {k: getattr(st, k) for k, _ in Stats._fields_}

    def reset_stats(self, timing: bool = False):
        self._check(_lib.nsrgs_reset_stats(self._h, int(timing)))
