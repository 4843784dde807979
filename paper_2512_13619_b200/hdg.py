"""Host-side mirror of the reference's operator API (namespace hdg, proj/include/hdg/*.hpp) on top of
the C ABI of include/hdgb200.h.  Names, argument meaning and error behaviour follow the reference:

    reference (C++)                         here
    --------------------------------------  ---------------------------------------------
    lu_invert_batch / gemm_batch / gemv_strided_batch (dense_batch.hpp)   same names
    make_case_setup (study.cpp:67-77)       Discretization.structured(...) + make_case_model(...)
    StateFields, compute_q (local_ops.hpp)  State, compute_q
    assemble_element_operators / assemble_residual / recover_local / gather_element_trace
    assemble_global, block_matvec, gather_extended, write_matrix / read_matrix (face_matrix.hpp)
    build_preconditioner, apply_base, apply_preconditioner, leja_order (preconditioner.hpp)
    gmres_solve (gmres.hpp), newton_solve / time_march (newton.hpp)
    hdg::Error hierarchy (errors.hpp)       HdgError and subclasses

Vectors may be numpy float64 arrays (host; staged by the library), raw device addresses (int) or
any object with data_ptr() (e.g. a torch CUDA tensor) for device-resident calls.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

__all__ = [
    "HdgError", "SingularBlock", "SingularMass", "SingularLocalSolve", "NonFiniteState", "NaNDetected",
    "LineSearchFailed", "DimensionMismatch", "InconsistentDimensions", "TooLargeForDense", "IoError",
    "InvalidMesh", "Unsupported", "CudaError",
    "Context", "Discretization", "Model", "State", "ElementOperators", "FaceBlockMatrix", "Preconditioner",
    "GmresConfig", "GmresStats", "NewtonConfig", "PrecondSpec", "SolveReport",
    "lu_invert_batch", "gemm_batch", "gemv_strided_batch", "compute_q", "assemble_element_operators",
    "assemble_residual", "gather_element_trace", "recover_local", "assemble_global", "block_matvec",
    "gather_extended", "write_matrix", "read_matrix", "build_preconditioner", "leja_order",
    "build_bj", "apply_bj", "build_asm", "apply_asm", "compute_harmonic_ritz", "apply_poly", "gmres_solve_fn",
    "precond_from_host", "ops_from_host",
    "harmonic_ritz_from_hessenberg", "gmres_solve", "orthogonalize", "newton_solve", "time_march",
    "make_case_model", "make_initial_state", "library_path", "load_library", "random_vector", "set_tuning",
    "SHAPES", "MODELS", "PRECONDS",
]

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "lib" / "libhdgb200.so"


def library_path() -> Path:
    return _LIB_PATH


# ---- errors (errors.hpp) --------------------------------------------------------------------------
class HdgError(RuntimeError):
    def __init__(self, msg, index=-1):
        super().__init__(msg)
        self.index = index


class SingularBlock(HdgError): pass
class SingularMass(SingularBlock): pass
class SingularLocalSolve(SingularBlock): pass
class NonFiniteState(HdgError): pass
class NaNDetected(HdgError): pass
class LineSearchFailed(HdgError): pass
class DimensionMismatch(HdgError): pass
class InconsistentDimensions(HdgError): pass
class TooLargeForDense(HdgError): pass
class IoError(HdgError): pass
class InvalidMesh(HdgError): pass
class Unsupported(HdgError): pass
class CudaError(HdgError): pass


_STATUS = {1: HdgError, 2: SingularBlock, 3: SingularMass, 4: SingularLocalSolve, 5: NonFiniteState,
           6: NaNDetected, 7: LineSearchFailed, 8: DimensionMismatch, 9: InconsistentDimensions,
           10: TooLargeForDense, 11: IoError, 12: InvalidMesh, 13: Unsupported, 14: CudaError}

SHAPES = {"quad": 0, "hex": 1, "tri": 2, "tet": 3}
MODELS = {"poisson": 0, "burgers": 1, "convdiff": 2, "elasticity": 3, "reaction": 4, "navier_stokes": 5}
PRECONDS = {"none": 0, "identity": 0, "bj": 1, "asm": 2, "ras": 3}
POLYS = {"gmres": 0, "chebyshev": 1}

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class _Dims(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("dim", "shape", "degree", "n_comp", "ne", "nf", "n_lfe", "n_orient",
                                       "pe", "pf", "qe", "qf", "nv")]


class _Time(C.Structure):
    _fields_ = [("dt", C.c_double), ("u_prev", _vp)]


class GmresConfig(C.Structure):
    """gmres.hpp:11-17"""
    _fields_ = [("restart", C.c_int), ("tol", C.c_double), ("max_iters", C.c_int), ("orth", C.c_int),
                ("track_diagnostics", C.c_int)]

    def __init__(self, restart=50, tol=1e-6, max_iters=1000, orth="cgs", track_diagnostics=False):
        super().__init__(restart, tol, max_iters, 1 if orth in ("mgs", 1, True) else 0, int(track_diagnostics))


class GmresStats(C.Structure):
    """gmres.hpp:19-34"""
    _fields_ = [("iters", C.c_int), ("restarts", C.c_int), ("final_rel_residual", C.c_double),
                ("t_mv", C.c_double), ("t_prec", C.c_double), ("t_orth", C.c_double), ("converged", C.c_int),
                ("max_orth_error", C.c_double), ("max_residual_gap", C.c_double)]
    residual_trace = None


class NewtonConfig(C.Structure):
    """newton.hpp:14-20 (dt / n_steps are arguments of time_march here)"""
    _fields_ = [("tol", C.c_double), ("max_newton", C.c_int), ("min_alpha", C.c_double)]

    def __init__(self, tol=1e-8, max_newton=50, min_alpha=1.0 / 1024.0):
        super().__init__(tol, max_newton, min_alpha)


class PrecondSpec(C.Structure):
    """newton.hpp:24-29 (+ poly_kind: 'gmres' harmonic-Ritz polynomial | 'chebyshev')"""
    _fields_ = [("kind", C.c_int), ("poly_degree", C.c_int), ("ritz_seed", C.c_uint64),
                ("ritz_per_restart", C.c_int), ("poly_kind", C.c_int)]

    def __init__(self, kind="bj", poly_degree=0, ritz_seed=12345, ritz_per_restart=False, poly_kind="gmres"):
        k = PRECONDS[kind] if isinstance(kind, str) else int(kind)
        pk = POLYS[poly_kind] if isinstance(poly_kind, str) else int(poly_kind)
        super().__init__(k, poly_degree, ritz_seed, int(ritz_per_restart), pk)


_MAXH = 128


class _Report(C.Structure):
    _fields_ = [("n_newton", C.c_int), ("n_gmres_total", C.c_int64), ("n_inner_prec_ops", C.c_int64),
                ("final_residual", C.c_double), ("converged", C.c_int),
                ("t_ass", C.c_double), ("t_mv", C.c_double), ("t_prec", C.c_double), ("t_orth", C.c_double),
                ("t_total", C.c_double), ("n_history", C.c_int),
                ("residual_history", C.c_double * (_MAXH + 1)), ("gmres_per_newton", C.c_int * _MAXH),
                ("alpha_history", C.c_double * _MAXH)]


class SolveReport:
    """newton.hpp:31-47"""

    def __init__(self, r: _Report):
        self.n_newton = r.n_newton
        self.n_gmres_total = r.n_gmres_total
        self.n_inner_prec_ops = r.n_inner_prec_ops
        self.final_residual = r.final_residual
        self.converged = bool(r.converged)
        self.t_ass, self.t_mv, self.t_prec, self.t_orth, self.t_total = r.t_ass, r.t_mv, r.t_prec, r.t_orth, r.t_total
        self.residual_history = list(r.residual_history[: r.n_history])
        k = min(r.n_newton, _MAXH)
        self.gmres_per_newton = list(r.gmres_per_newton[:k])
        self.alpha_history = [a for a in r.alpha_history[:k] if a != 0.0]

    def __repr__(self):
        return (f"SolveReport(n_newton={self.n_newton}, n_gmres_total={self.n_gmres_total}, "
                f"final_residual={self.final_residual:.6e}, converged={self.converged})")


# hdgb_op_fn: int (*)(void* user, const double* in, double* out, int64_t n) on DEVICE vectors
OP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)

_lib = None


def load_library():
    """Loads libhdgb200.so; fails loudly when it has not been built (no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise FileNotFoundError(f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                                f"g.build()'` or `make -C paper_2512_13619_b200/csrc` (there is no CPU fallback)")
    L = C.CDLL(str(_LIB_PATH))
    i, d, u64, i64, cp = C.c_int, C.c_double, C.c_uint64, C.c_int64, C.c_char_p
    pp = C.POINTER(_vp)
    sig = {
        "hdgb_ctx_create": (i, [i, pp]), "hdgb_ctx_destroy": (None, [_vp]), "hdgb_last_error": (cp, [_vp]),
        "hdgb_last_error_index": (i64, [_vp]), "hdgb_ctx_set_stream": (i, [_vp, _vp]), "hdgb_ctx_stream": (_vp, [_vp]),
        "hdgb_ctx_synchronize": (i, [_vp]), "hdgb_ctx_launch_count": (i64, [_vp]),
        "hdgb_ctx_reset_launch_count": (None, [_vp]), "hdgb_version": (cp, []),
        "hdgb_set_tuning": (i, [cp, i64]),
        "hdgb_pool_stats": (None, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "hdgb_lu_invert_batch": (i, [_vp, i, i, _vp, _vp]),
        "hdgb_gemm_batch": (i, [_vp, i, i, i, _vp, i, i, i, _vp, i, _vp]),
        "hdgb_gemv_strided_batch": (i, [_vp, i, i, i, _vp, _vp, _vp, i]),
        "hdgb_disc_create_structured": (i, [_vp, i, i, i, i, i, _dp, _dp, d, u64, pp]),
        "hdgb_disc_create_from_mesh": (i, [_vp, i, i, i, i, i, i, _vp, _vp, pp]),
        "hdgb_disc_destroy": (None, [_vp]), "hdgb_disc_dims": (i, [_vp, C.POINTER(_Dims)]),
        "hdgb_disc_get_f64": (i, [_vp, cp, _vp, i64, C.POINTER(i64)]),
        "hdgb_disc_get_i32": (i, [_vp, cp, _vp, i64, C.POINTER(i64)]),
        "hdgb_disc_set_boundary_tags": (i, [_vp, _vp]),
        "hdgb_model_create": (i, [_vp, _vp, i, _vp, i, _vp, _vp, pp]), "hdgb_model_destroy": (None, [_vp]),
        "hdgb_state_create": (i, [_vp, _vp, pp]), "hdgb_state_destroy": (None, [_vp]),
        "hdgb_state_set": (i, [_vp, cp, _vp]), "hdgb_state_get": (i, [_vp, cp, _vp]),
        "hdgb_state_ptr": (_vp, [_vp, cp]),
        "hdgb_compute_q": (i, [_vp, _vp]),
        "hdgb_assemble_element_operators": (i, [_vp, _vp, _vp, C.POINTER(_Time), i, pp]),
        "hdgb_ops_destroy": (None, [_vp]), "hdgb_ops_get": (i, [_vp, cp, _vp, i64, C.POINTER(i64)]),
        "hdgb_ops_ptr": (_vp, [_vp, cp]),
        "hdgb_assemble_residual": (i, [_vp, _vp, _vp, C.POINTER(_Time), _vp, _vp, _dp]),
        "hdgb_gather_element_trace": (i, [_vp, _vp, _vp]), "hdgb_recover_local": (i, [_vp, _vp, _vp, _vp]),
        "hdgb_assemble_global": (i, [_vp, _vp, pp, _vp]),
        "hdgb_matrix_create": (i, [_vp, i, i, i, i, _vp, _vp, pp]), "hdgb_matrix_destroy": (None, [_vp]),
        "hdgb_matrix_dims": (i, [_vp, C.POINTER(i)]), "hdgb_matrix_get_neighbor": (i, [_vp, _vp]),
        "hdgb_matrix_get_blocks": (i, [_vp, _vp]), "hdgb_matrix_blocks_ptr": (_vp, [_vp]),
        "hdgb_matrix_rhs": (_vp, [_vp]), "hdgb_block_matvec": (i, [_vp, _vp, _vp]),
        "hdgb_gather_extended": (i, [_vp, _vp, _vp]), "hdgb_matrix_write": (i, [_vp, _vp, cp]),
        "hdgb_matrix_read": (i, [_vp, cp, pp, _vp]),
        "hdgb_precond_spec_default": (None, [C.POINTER(PrecondSpec)]),
        "hdgb_build_preconditioner": (i, [_vp, _vp, _vp, C.POINTER(PrecondSpec), pp]),
        "hdgb_precond_destroy": (None, [_vp]), "hdgb_precond_get": (i, [_vp, cp, _vp, i64, C.POINTER(i64)]),
        "hdgb_precond_set_ritz": (i, [_vp, _vp, i]), "hdgb_precond_apply_base": (i, [_vp, _vp, _vp]),
        "hdgb_precond_apply": (i, [_vp, _vp, _vp, _vp]), "hdgb_precond_inner_ops": (i64, [_vp]),
        "hdgb_leja_order": (i, [_vp, i, _vp, C.POINTER(i)]),
        "hdgb_harmonic_ritz_from_hessenberg": (i, [_vp, i, i, _vp, C.POINTER(i)]),
        "hdgb_gmres_config_default": (None, [C.POINTER(GmresConfig)]),
        "hdgb_gmres_solve": (i, [_vp, _vp, _vp, _vp, C.POINTER(GmresConfig), _vp, C.POINTER(GmresStats), _vp]),
        "hdgb_orthogonalize": (i, [_vp, _vp, i, i64, _vp, i, _vp]),
        "hdgb_ctx_enable_phase_timing": (None, [_vp, i]),
        "hdgb_newton_config_default": (None, [C.POINTER(NewtonConfig)]),
        "hdgb_newton_solve": (i, [_vp, _vp, _vp, C.POINTER(NewtonConfig), C.POINTER(GmresConfig),
                                  C.POINTER(PrecondSpec), C.POINTER(_Time), C.POINTER(_Report)]),
        "hdgb_time_march": (i, [_vp, _vp, _vp, d, i, C.POINTER(NewtonConfig), C.POINTER(GmresConfig),
                                C.POINTER(PrecondSpec), C.POINTER(_Report)]),
        "hdgb_disc_create_from_tables": (i, [_vp, i, i, i, i, i, i, i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, i, i, _vp, i64, pp]),
        "hdgb_mesh_connectivity": (i, [i, i, i, _vp, _vp, pp]),
        "hdgb_comm_nccl_unique_id": (i, [_vp]), "hdgb_comm_create_nccl": (i, [_vp, _vp, i, i]),
        "hdgb_comm_set_halo_plan": (i, [_vp, i, _vp, _vp, _vp, _vp, _vp]),
        "hdgb_comm_set_callbacks": (i, [_vp, i, i, _vp, _vp, _vp]), "hdgb_comm_destroy": (None, [_vp]),
        "hdgb_halo_exchange": (i, [_vp, _vp, i]), "hdgb_halo_exchange_begin": (i, [_vp, _vp, i]),
        "hdgb_halo_exchange_end": (i, [_vp]), "hdgb_allreduce_sum": (i, [_vp, _vp, i]),
        "hdgb_comm_rank": (i, [_vp]), "hdgb_comm_size": (i, [_vp]),
        "hdgb_device_alloc": (i, [_vp, i64, pp]), "hdgb_device_free": (None, [_vp, _vp]),
        "hdgb_copy": (i, [_vp, _vp, _vp, i64]),
        "hdgb_ops_create": (i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, pp]),
        "hdgb_build_bj": (i, [_vp, pp]), "hdgb_apply_bj": (i, [_vp, _vp, _vp]),
        "hdgb_build_asm": (i, [_vp, _vp, pp]), "hdgb_apply_asm": (i, [_vp, _vp, _vp]),
        "hdgb_precond_create": (i, [_vp, i, i, i, _vp, _vp, _vp, i, pp]),
        "hdgb_compute_harmonic_ritz": (i, [_vp, OP_FN, _vp, i64, i, u64, _vp, C.POINTER(i)]),
        "hdgb_apply_poly": (i, [_vp, OP_FN, _vp, _vp, _vp, _vp, C.POINTER(i64)]),
        "hdgb_gmres_solve_fn": (i, [_vp, i64, OP_FN, _vp, OP_FN, _vp, _vp, _vp, C.POINTER(GmresConfig), _vp,
                                    C.POINTER(GmresStats), _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)  # AttributeError = the library does not export what the header declares
        fn.restype = res
        fn.argtypes = args
    L._signatures = sig
    _lib = L
    return L


def set_tuning(key: str, value: int):
    """Kernel-selection knobs (hdgb_set_tuning): 'use_stream', 'stream_min_elems'."""
    if load_library().hdgb_set_tuning(key.encode(), int(value)) != 0:
        raise KeyError(key)


def pool_stats():
    """(cudaMalloc calls, cudaFree calls) issued by the caching allocator so far."""
    a, f = C.c_int64(0), C.c_int64(0)
    load_library().hdgb_pool_stats(C.byref(a), C.byref(f))
    return a.value, f.value


def exported_symbols():
    """The entry points include/hdgb200.h declares (used by the CPU-side ABI test)."""
    return sorted(load_library()._signatures)


def _ptr(a):
    """numpy array -> host address; int -> device address; object with data_ptr() -> its address."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "arrays must be contiguous"
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return int(a)


def _f64(a):
    if isinstance(a, np.ndarray) or isinstance(a, (list, tuple)):
        return np.ascontiguousarray(a, dtype=np.float64)
    return a


def random_vector(n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """The reference tests' generator: scale * (2*((mt19937_64()>>11)*2^-53) - 1) (test_helpers.hpp:11-16)."""
    # numpy's MT19937 is the 32-bit variant, so the 64-bit engine is restated here.
    mt = _MT19937_64(seed)
    out = np.empty(n)
    for k in range(n):
        out[k] = scale * (2.0 * ((mt.next() >> 11) * 2.0 ** -53) - 1.0)
    return out


class _MT19937_64:
    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def next(self):
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


class Context:
    """Device, stream, workspaces and the last error (hdgb_ctx)."""

    def __init__(self, device: int = 0):
        self._L = load_library()
        h = _vp()
        st = self._L.hdgb_ctx_create(device, C.byref(h))
        if st != 0:
            raise _STATUS.get(st, HdgError)("no usable CUDA device: this library has no CPU fallback")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._L.hdgb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, status: int):
        if status != 0:
            msg = self._L.hdgb_last_error(self._h).decode()
            raise _STATUS.get(status, HdgError)(msg, self._L.hdgb_last_error_index(self._h))

    def synchronize(self):
        self.check(self._L.hdgb_ctx_synchronize(self._h))

    def set_stream(self, cuda_stream: int):
        self.check(self._L.hdgb_ctx_set_stream(self._h, cuda_stream))

    @property
    def stream(self) -> int:
        return self._L.hdgb_ctx_stream(self._h) or 0

    @property
    def launch_count(self) -> int:
        return self._L.hdgb_ctx_launch_count(self._h)

    def reset_launch_count(self):
        self._L.hdgb_ctx_reset_launch_count(self._h)

    def enable_phase_timing(self, on=True):
        self._L.hdgb_ctx_enable_phase_timing(self._h, int(on))

    def alloc(self, n: int) -> int:
        p = _vp()
        self.check(self._L.hdgb_device_alloc(self._h, n, C.byref(p)))
        return p.value

    def free(self, p: int):
        self._L.hdgb_device_free(self._h, p)

    def copy(self, dst, src, n: int):
        self.check(self._L.hdgb_copy(self._h, _ptr(dst), _ptr(src), n))


# ---- dense batch kernels (dense_batch.hpp:36-51) ---------------------------------------------------
def lu_invert_batch(ctx: Context, a, n: int, batch: int) -> np.ndarray:
    a = _f64(a)
    out = np.empty(n * n * batch)
    ctx.check(ctx._L.hdgb_lu_invert_batch(ctx._h, n, batch, _ptr(a), _ptr(out)))
    return out


def gemm_batch(ctx: Context, a, ar, ac, abatch, b, br, bc, bbatch, transpose_a=False) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    m = ac if transpose_a else ar
    out = np.empty(max(abatch, bbatch) * m * bc)
    ctx.check(ctx._L.hdgb_gemm_batch(ctx._h, ar, ac, abatch, _ptr(a), br, bc, bbatch, _ptr(b), int(transpose_a), _ptr(out)))
    return out


def gemv_strided_batch(ctx: Context, a, rows, cols, batch, x, y=None, accumulate=False) -> np.ndarray:
    a, x = _f64(a), _f64(x)
    yv = np.zeros(rows * batch) if y is None else _f64(y).copy()
    ctx.check(ctx._L.hdgb_gemv_strided_batch(ctx._h, rows, cols, batch, _ptr(a), _ptr(x), _ptr(yv), int(accumulate)))
    return yv


# ---- discretisation --------------------------------------------------------------------------------
class Discretization:
    """Mesh + master element + geometry + local factors (Mesh2D, BasisTab, GeomFactors, LocalFactors)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self._h = handle
        self._L = load_library()
        d = _Dims()
        self._L.hdgb_disc_dims(handle, C.byref(d))
        for n, _ in _Dims._fields_:
            setattr(self, n, getattr(d, n))
        self.npe = self.n_comp * self.pe
        self.mpf = self.n_comp * self.pf
        self.nfl = self.n_lfe * self.mpf
        self.nb = 2 * self.n_lfe - 1
        self.n_dof = self.mpf * self.nf

    @classmethod
    def structured(cls, ctx: Context, shape="quad", n=8, degree=2, n_comp=1, quad_points=0, lo=None, hi=None,
                   jitter=0.0, seed=12345):
        """build_structured_quad + gauss_rule(k+2) + tabulate_basis + compute_geometry +
        precompute_local_factors (study.cpp:67-77); hex analogue for shape='hex'."""
        h = _vp()
        lo_a = None if lo is None else (C.c_double * 3)(*(list(lo) + [0.0] * 3)[:3])
        hi_a = None if hi is None else (C.c_double * 3)(*(list(hi) + [1.0] * 3)[:3])
        if ctx is None:
            # host-only tables (mesh / master element / geometry); operators need a Context
            st = load_library().hdgb_disc_create_structured(None, SHAPES[shape], n, degree, n_comp, quad_points, lo_a,
                                                            hi_a, jitter, seed, C.byref(h))
            if st != 0:
                raise _STATUS.get(st, HdgError)(f"host-only discretisation failed (status {st})")
            return cls(None, h)
        ctx.check(ctx._L.hdgb_disc_create_structured(ctx._h, SHAPES[shape], n, degree, n_comp, quad_points, lo_a, hi_a,
                                                     jitter, seed, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_mesh(cls, ctx: Context, shape, degree, elem_verts, vertex_coords, n_comp=1, quad_points=0):
        ev = np.ascontiguousarray(elem_verts, dtype=np.int32)
        vc = np.ascontiguousarray(vertex_coords, dtype=np.float64)
        h = _vp()
        ctx.check(ctx._L.hdgb_disc_create_from_mesh(ctx._h, SHAPES[shape], degree, n_comp, quad_points, ev.shape[0],
                                                    vc.shape[0], _ptr(ev), _ptr(vc), C.byref(h)))
        return cls(ctx, h)

    def close(self):
        if getattr(self, "_h", None):
            self._L.hdgb_disc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def table(self, name: str) -> np.ndarray:
        n = C.c_int64()
        L = self._L
        st = L.hdgb_disc_get_f64(self._h, name.encode(), None, 0, C.byref(n))
        if st == 0:
            out = np.empty(n.value)
            if L.hdgb_disc_get_f64(self._h, name.encode(), _ptr(out), n.value, C.byref(n)) != 0:
                raise HdgError(f"table {name}")
            return out
        st = L.hdgb_disc_get_i32(self._h, name.encode(), None, 0, C.byref(n))
        if st != 0:
            raise KeyError(name)
        out = np.empty(n.value, dtype=np.int32)
        if L.hdgb_disc_get_i32(self._h, name.encode(), _ptr(out), n.value, C.byref(n)) != 0:
            raise HdgError(f"table {name}")
        return out

    def set_boundary_tags(self, tags):
        t = np.ascontiguousarray(tags, dtype=np.int32)
        self.ctx.check(self.ctx._L.hdgb_disc_set_boundary_tags(self._h, _ptr(t)))

    # -- nodal interpolation helpers (interpolate_volume / interpolate_trace, local_ops.cpp:462-495)
    def volume_node_coords(self) -> np.ndarray:
        """(ne, pe, dim) physical coordinates of the element nodes."""
        D = self.dim
        vc = self.table("vertex_coords").reshape(-1, D)
        ev = self.table("element_vertices").reshape(self.ne, -1)
        v = vc[ev]  # ne, vpe, D
        xi = self.table("elem_nodes").reshape(self.pe, D)
        if self.shape in (SHAPES["tri"], SHAPES["tet"]):
            N = np.concatenate([1.0 - xi.sum(axis=1, keepdims=True), xi], axis=1)      # barycentric, affine map
        elif D == 2:
            a, b = xi[:, 0], xi[:, 1]
            N = np.stack([(1 - a) * (1 - b), a * (1 - b), a * b, (1 - a) * b], axis=1)
        else:
            a, b, c = xi[:, 0], xi[:, 1], xi[:, 2]
            cs = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
            N = np.stack([(a if s[0] else 1 - a) * (b if s[1] else 1 - b) * (c if s[2] else 1 - c) for s in cs], axis=1)
        return np.einsum("pc,ecd->epd", N, v)

    def trace_node_coords(self) -> np.ndarray:
        """(nf, pf, dim) physical coordinates of the face nodes in canonical face order."""
        D = self.dim
        vc = self.table("vertex_coords").reshape(-1, D)
        fv = self.table("face_vertices").reshape(self.nf, -1)
        v = vc[fv]
        fn = self.table("face_nodes").reshape(self.pf, D - 1)
        if D == 2:
            t = fn[:, 0]
            return v[:, None, 0, :] + t[None, :, None] * (v[:, None, 1, :] - v[:, None, 0, :])
        s, t = fn[:, 0], fn[:, 1]
        if self.shape == SHAPES["tet"]:
            N = np.stack([1 - s - t, s, t], axis=1)
        else:
            N = np.stack([(1 - s) * (1 - t), s * (1 - t), s * t, (1 - s) * t], axis=1)
        return np.einsum("pc,fcd->fpd", N, v)

    def interpolate_volume(self, fn) -> np.ndarray:
        """fn(x: (..., dim)) -> (..., M) or (...); returns u in the state layout [e][m][i]."""
        x = self.volume_node_coords()
        val = np.asarray(fn(x), dtype=np.float64)
        if val.ndim == 2:
            val = val[..., None]
        val = np.broadcast_to(val, (self.ne, self.pe, self.n_comp))
        return np.ascontiguousarray(val.transpose(0, 2, 1)).ravel()

    def interpolate_trace(self, fn) -> np.ndarray:
        x = self.trace_node_coords()
        val = np.asarray(fn(x), dtype=np.float64)
        if val.ndim == 2:
            val = val[..., None]
        val = np.broadcast_to(val, (self.nf, self.pf, self.n_comp))
        return np.ascontiguousarray(val.transpose(0, 2, 1)).ravel()

    def quad_coords(self):
        """((ne, qe, dim), (nf, qf, dim)) physical quadrature point coordinates."""
        if getattr(self, "_quad_coords", None) is None:  # geometry is immutable: fetch the tables once
            self._quad_coords = (self.table("elem_coords").reshape(self.ne, self.qe, self.dim),
                                 self.table("face_coords").reshape(self.nf, self.qf, self.dim))
        return self._quad_coords

    def l2_error(self, u, exact) -> float:
        """L2 error of component-wise nodal coefficients u against exact(x) at the assembly
        quadrature points (the reference's l2_error uses a finer rule, local_ops.cpp:498-517)."""
        phi = self.table("phi").reshape(self.qe, self.pe)
        w = self.table("elem_weights")
        det = self.table("elem_detjac").reshape(self.ne, self.qe)
        xq, _ = self.quad_coords()
        uu = np.asarray(u).reshape(self.ne, self.n_comp, self.pe)
        uh = np.einsum("gi,emi->egm", phi, uu)
        ex = np.asarray(exact(xq), dtype=np.float64)
        if ex.ndim == 2:
            ex = ex[..., None]
        diff = uh - ex
        return float(np.sqrt(np.einsum("g,eg,egm->", w, det, diff * diff)))


class Model:
    """PdeModel (models.hpp:27-50) as a device functor tag + parameters + tabulated x-only data."""

    def __init__(self, disc: Discretization, kind: str, params, forcing=None, dirichlet=None, exact=None,
                 initial=None, name=None, forcing_q=None, dirichlet_q=None):
        """forcing / dirichlet: callables of x, tabulated here at the quadrature points; forcing_q / dirichlet_q:
        the same data already tabulated ([e][g][m] / [f][g][m] host arrays), uploaded as they are.  On a host-only
        discretisation (ctx None) the model is a description only (used to feed the CPU oracle)."""
        self.disc, self.kind, self.params = disc, kind, list(params)
        self.exact_solution, self.initial_state, self.name = exact, initial, name or kind
        self._forcing, self._dirichlet = forcing, dirichlet
        ctx = disc.ctx
        fq, dq = forcing_q, dirichlet_q
        if (forcing is not None and fq is None) or (dirichlet is not None and dq is None):
            xq, xf = disc.quad_coords()
            if forcing is not None and fq is None:
                fq = np.asarray(forcing(xq), dtype=np.float64)
                fq = np.ascontiguousarray(np.broadcast_to(fq.reshape(disc.ne, disc.qe, -1), (disc.ne, disc.qe, disc.n_comp)))
            if dirichlet is not None and dq is None:
                dq = np.asarray(dirichlet(xf), dtype=np.float64)
                dq = np.ascontiguousarray(np.broadcast_to(dq.reshape(disc.nf, disc.qf, -1), (disc.nf, disc.qf, disc.n_comp)))
        self.forcing_q, self.dirichlet_q = fq, dq
        self._h = None
        if ctx is None:
            return
        p = np.asarray(self.params, dtype=np.float64)
        h = _vp()
        ctx.check(ctx._L.hdgb_model_create(ctx._h, disc._h, MODELS[kind], _ptr(p), len(p), _ptr(_f64(fq)), _ptr(_f64(dq)), C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self.disc.ctx._L.hdgb_model_destroy(self._h)
                self._h = None
        except Exception:
            pass


def make_case_model(disc: Discretization, case: str, tau=None, nu=1.0 / 200.0, kappa=1.0, velocity=(0.0, 1.0),
                    lam=1.0, mu=1.0, alpha=1.0) -> Model:
    # (mu doubles as the dynamic viscosity of the Navier-Stokes case)
    """make_case_model (study.cpp:31-65) plus the 3D / multi-component cases of BASELINE.json."""
    pi = np.pi
    D = disc.dim

    def sinprod(x):
        return np.prod(np.sin(pi * x), axis=-1)

    if case in ("poisson2d", "poisson3d", "poisson"):
        return Model(disc, "poisson", [1.0 if tau is None else tau], forcing=lambda x: D * pi * pi * sinprod(x),
                     dirichlet=sinprod, exact=sinprod, name=case)
    if case in ("heat2d", "heat"):
        return Model(disc, "poisson", [1.0 if tau is None else tau], initial=sinprod, name=case)
    if case in ("burgers2d", "burgers"):
        return Model(disc, "burgers", [nu, (10.0 * nu + 1.0) if tau is None else tau],
                     initial=lambda x: 1.0 - 2.0 * x[..., 0], name=case)
    if case in ("convdiff2d", "convdiff"):
        c = list(velocity) + [0.0] * (3 - len(velocity))

        def forcing(x):
            s, co = np.sin(pi * x), np.cos(pi * x)
            conv = 0.0
            for d in range(D):
                term = co[..., d]
                for e in range(D):
                    if e != d:
                        term = term * s[..., e]
                conv = conv + c[d] * term
            return pi * conv + D * kappa * pi * pi * np.prod(s, axis=-1)
        return Model(disc, "convdiff", c + [kappa, -1.0 if tau is None else tau], forcing=forcing, dirichlet=sinprod,
                     exact=sinprod, name=case)
    if case in ("reaction2d", "reaction"):
        return Model(disc, "reaction", [1.0 if tau is None else tau, alpha],
                     forcing=lambda x: D * pi * pi * sinprod(x) + alpha * sinprod(x) ** 3, dirichlet=sinprod,
                     exact=sinprod, name=case)
    if case in ("elasticity", "elasticity2d", "elasticity3d"):
        # manufactured displacement u_m = sin(pi x_0)...sin(pi x_{D-1}) * (m+1), clamped everywhere
        def exact(x):
            return np.stack([(m + 1.0) * sinprod(x) for m in range(D)], axis=-1)

        def forcing(x):
            # f = -div sigma, sigma = mu (grad u + grad u^T) + lam tr(grad u) I
            s, co = np.sin(pi * x), np.cos(pi * x)
            P = np.prod(s, axis=-1)

            def d2(m, a, b):  # d^2 u_m / dx_a dx_b
                if a == b:
                    return -(m + 1.0) * pi * pi * P
                t = co[..., a] * co[..., b]
                for e in range(D):
                    if e not in (a, b):
                        t = t * s[..., e]
                return (m + 1.0) * pi * pi * t
            out = []
            for m in range(D):
                acc = 0.0
                for d in range(D):
                    acc = acc + mu * (d2(m, d, d) + d2(d, m, d)) + lam * d2(d, d, m)
                out.append(-acc)
            return np.stack(out, axis=-1)
        return Model(disc, "elasticity", [lam, mu, 1.0 if tau is None else tau, 0.0], forcing=forcing,
                     dirichlet=exact, exact=exact, name=case)
    if case in ("navier_stokes", "ns", "taylor_green"):
        # compressible Navier-Stokes, conservative variables (rho, rho v, rho E); the initial / boundary
        # state is a smooth low-Mach vortex field of Taylor-Green type on the unit box (PAPER.md 5.7)
        gamma, pr = 1.4, 0.71
        mach = 0.1
        p0 = 1.0 / (gamma * mach * mach)

        def state(x):
            X = [2 * pi * x[..., d] for d in range(D)]
            if D == 2:
                v = [np.sin(X[0]) * np.cos(X[1]), -np.cos(X[0]) * np.sin(X[1])]
                p = p0 + 0.25 * (np.cos(2 * X[0]) + np.cos(2 * X[1]))
            else:
                v = [np.sin(X[0]) * np.cos(X[1]) * np.cos(X[2]), -np.cos(X[0]) * np.sin(X[1]) * np.cos(X[2]), 0.0 * X[0]]
                p = p0 + (np.cos(2 * X[0]) + np.cos(2 * X[1])) * (np.cos(2 * X[2]) + 2.0) / 16.0
            rho = np.ones_like(X[0])
            rhoE = p / (gamma - 1.0) + 0.5 * rho * sum(vi * vi for vi in v)
            return np.stack([rho] + [rho * vi for vi in v] + [rhoE], axis=-1)
        return Model(disc, "navier_stokes", [gamma, mu, pr, (1.0 / mach + 1.0) if tau is None else tau], dirichlet=state,
                     initial=state, name=case)
    raise HdgError(f"unknown case '{case}'")


# ---- state -----------------------------------------------------------------------------------------
class State:
    """StateFields (local_ops.hpp:16-23) on the device."""

    def __init__(self, disc: Discretization):
        self.disc = disc
        h = _vp()
        disc.ctx.check(disc.ctx._L.hdgb_state_create(disc.ctx._h, disc._h, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self.disc.ctx._L.hdgb_state_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def _size(self, name):
        return self.disc.n_dof if name == "uhat" else self.disc.npe * self.disc.ne

    def set(self, name: str, v):
        v = _f64(v)
        if isinstance(v, np.ndarray) and v.size != self._size(name):
            raise DimensionMismatch(f"state field {name}: expected {self._size(name)} values, got {v.size}")
        self.disc.ctx.check(self.disc.ctx._L.hdgb_state_set(self._h, name.encode(), _ptr(v)))

    def get(self, name: str) -> np.ndarray:
        out = np.empty(self._size(name))
        self.disc.ctx.check(self.disc.ctx._L.hdgb_state_get(self._h, name.encode(), _ptr(out)))
        return out

    def ptr(self, name: str) -> int:
        return self.disc.ctx._L.hdgb_state_ptr(self._h, name.encode())

    u = property(lambda s: s.get("u"), lambda s, v: s.set("u", v))
    uhat = property(lambda s: s.get("uhat"), lambda s, v: s.set("uhat", v))

    def q(self, d: int) -> np.ndarray:
        return self.get(f"q{d}")


def make_initial_state(disc: Discretization, model: Model) -> State:
    """make_initial_state (study.cpp:79-92)."""
    s = State(disc)
    if model.initial_state is not None:
        s.u = disc.interpolate_volume(model.initial_state)
        s.uhat = disc.interpolate_trace(model.initial_state)
    compute_q(disc, s)
    return s


def _time(dt, u_prev):
    if dt is None or not (dt > 0.0):
        return None, None
    keep = _f64(u_prev)
    return _Time(dt, _ptr(keep)), keep


def compute_q(disc: Discretization, state: State):
    disc.ctx.check(disc.ctx._L.hdgb_compute_q(disc._h, state._h))


class ElementOperators:
    """ElementOperators (local_ops.hpp:30-61) on the device."""

    def __init__(self, disc, handle):
        self.disc, self._h = disc, handle

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self.disc.ctx._L.hdgb_ops_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def get(self, name: str) -> np.ndarray:
        n = C.c_int64()
        L, ctx = self.disc.ctx._L, self.disc.ctx
        ctx.check(L.hdgb_ops_get(self._h, name.encode(), None, 0, C.byref(n)))
        out = np.empty(n.value)
        ctx.check(L.hdgb_ops_get(self._h, name.encode(), _ptr(out), n.value, C.byref(n)))
        return out

    def ptr(self, name: str) -> int:
        return self.disc.ctx._L.hdgb_ops_ptr(self._h, name.encode())


def assemble_element_operators(disc, model, state, dt=None, u_prev=None, keep_raw=False) -> ElementOperators:
    t, keep = _time(dt, u_prev)
    h = _vp()
    disc.ctx.check(disc.ctx._L.hdgb_assemble_element_operators(disc._h, model._h, state._h,
                                                               C.byref(t) if t else None, int(keep_raw), C.byref(h)))
    return ElementOperators(disc, h)


def assemble_residual(disc, model, state, dt=None, u_prev=None):
    """Returns (trace, interior, stacked 2-norm) -- Residuals + residual_norm (local_ops.cpp:245-250,432-450)."""
    t, keep = _time(dt, u_prev)
    tr, it = np.empty(disc.n_dof), np.empty(disc.npe * disc.ne)
    nrm = C.c_double()
    disc.ctx.check(disc.ctx._L.hdgb_assemble_residual(disc._h, model._h, state._h, C.byref(t) if t else None,
                                                      _ptr(tr), _ptr(it), C.byref(nrm)))
    return tr, it, nrm.value


def gather_element_trace(disc, face_values) -> np.ndarray:
    v = _f64(face_values)
    out = np.empty(disc.nfl * disc.ne)
    disc.ctx.check(disc.ctx._L.hdgb_gather_element_trace(disc._h, _ptr(v), _ptr(out)))
    return out


def recover_local(disc, ops: ElementOperators, duhat) -> np.ndarray:
    """recover_local (local_ops.cpp:452-460); takes the FACE-major duhat (the element gather is fused)."""
    v = _f64(duhat)
    out = np.empty(disc.npe * disc.ne)
    disc.ctx.check(disc.ctx._L.hdgb_recover_local(disc._h, ops._h, _ptr(v), _ptr(out)))
    return out


# ---- global operator -------------------------------------------------------------------------------
class FaceBlockMatrix:
    """FaceBlockMatrix (face_matrix.hpp:26-43) on the device."""

    def __init__(self, ctx: Context, handle):
        self.ctx, self._h = ctx, handle
        d = (C.c_int * 4)()
        ctx._L.hdgb_matrix_dims(handle, d)
        self.m, self.pf, self.n_lfe, self.nf = list(d)
        self.nb = 2 * self.n_lfe - 1
        self.block_dim = self.m * self.pf
        self.n_dof = self.block_dim * self.nf      # owned unknowns (rows)
        self.n_vec = self.n_dof                    # vector length (incl. halo faces when partitioned)

    @classmethod
    def from_host(cls, ctx, m, pf, n_lfe, nf, neighbor, blocks):
        nb = np.ascontiguousarray(neighbor, dtype=np.int64)
        bl = _f64(blocks)
        h = _vp()
        ctx.check(ctx._L.hdgb_matrix_create(ctx._h, m, pf, n_lfe, nf, _ptr(nb), _ptr(bl), C.byref(h)))
        return cls(ctx, h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self.ctx._L.hdgb_matrix_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def neighbor(self) -> np.ndarray:
        out = np.empty(self.nf * self.nb, dtype=np.int64)
        self.ctx.check(self.ctx._L.hdgb_matrix_get_neighbor(self._h, _ptr(out)))
        return out

    @property
    def blocks(self) -> np.ndarray:
        out = np.empty(self.block_dim * self.block_dim * self.nb * self.nf)
        self.ctx.check(self.ctx._L.hdgb_matrix_get_blocks(self._h, _ptr(out)))
        return out

    @property
    def rhs(self) -> np.ndarray:
        out = np.empty(self.n_dof)
        p = self.ctx._L.hdgb_matrix_rhs(self._h)
        if not p:
            raise HdgError("matrix has no right-hand side")
        self.ctx.copy(out, p, self.n_dof)
        return out

    def rhs_ptr(self) -> int:
        return self.ctx._L.hdgb_matrix_rhs(self._h) or 0

    def blocks_ptr(self) -> int:
        return self.ctx._L.hdgb_matrix_blocks_ptr(self._h)

    def to_dense(self, limit=20000) -> np.ndarray:
        """to_dense (face_matrix.cpp:116-135), host-side expansion for tests."""
        if self.n_dof > limit:
            raise TooLargeForDense(f"dense expansion of {self.n_dof} unknowns refused")
        bd, nb = self.block_dim, self.nb
        blocks = self.blocks.reshape(self.nf, nb, bd, bd)  # [f][slot][c][r]
        nbr = self.neighbor.reshape(self.nf, nb)
        a = np.zeros((self.n_dof, self.n_dof))
        for f in range(self.nf):
            for s in range(nb):
                g = nbr[f, s]
                if g < 0:
                    continue
                a[f * bd:(f + 1) * bd, g * bd:(g + 1) * bd] += blocks[f, s].T
        return a


def assemble_global(disc, ops: ElementOperators):
    """assemble_global (face_matrix.cpp:11-61) -> (FaceBlockMatrix, rhs)."""
    h = _vp()
    rhs = np.empty(disc.n_dof)
    disc.ctx.check(disc.ctx._L.hdgb_assemble_global(disc._h, ops._h, C.byref(h), _ptr(rhs)))
    k = FaceBlockMatrix(disc.ctx, h)
    k.n_vec = disc.n_dof   # a partitioned discretisation spans owned + halo faces
    return k, rhs


def block_matvec(k: FaceBlockMatrix, x, y=None):
    x = _f64(x)
    if isinstance(x, np.ndarray) and x.size != k.n_vec:
        raise DimensionMismatch(f"block_matvec: vector has {x.size} entries, operator {k.n_vec}")
    out = np.empty(k.n_vec) if y is None else y
    k.ctx.check(k.ctx._L.hdgb_block_matvec(k._h, _ptr(x), _ptr(out)))
    return out


def gather_extended(k: FaceBlockMatrix, x) -> np.ndarray:
    x = _f64(x)
    out = np.empty(k.n_dof * k.nb)
    k.ctx.check(k.ctx._L.hdgb_gather_extended(k._h, _ptr(x), _ptr(out)))
    return out


def write_matrix(path, k: FaceBlockMatrix, rhs=None):
    r = _f64(rhs)
    k.ctx.check(k.ctx._L.hdgb_matrix_write(k._h, _ptr(r), os.fsencode(path)))


def read_matrix(ctx: Context, path):
    h = _vp()
    # header peek for the rhs size
    with open(path, "rb") as fp:
        head = fp.read(24)
    if len(head) == 24 and head[:4] == b"HDGK":
        m, pf, _, nf = np.frombuffer(head[8:24], dtype=np.uint32)
        rhs = np.empty(int(m) * int(pf) * int(nf))
    else:
        rhs = None
    ctx.check(ctx._L.hdgb_matrix_read(ctx._h, os.fsencode(path), C.byref(h), _ptr(rhs)))
    return FaceBlockMatrix(ctx, h), rhs


# ---- preconditioners -------------------------------------------------------------------------------
class Preconditioner:
    """Preconditioner (preconditioner.hpp:19-29) on the device."""

    def __init__(self, ctx, handle, k):
        self.ctx, self._h, self.k = ctx, handle, k

    @property
    def _n_vec(self):
        return self.k.n_vec if hasattr(self.k, "n_vec") else self.k.n_dof

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self.ctx._L.hdgb_precond_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def get(self, name) -> np.ndarray:
        n = C.c_int64()
        self.ctx.check(self.ctx._L.hdgb_precond_get(self._h, name.encode(), None, 0, C.byref(n)))
        out = np.empty(n.value)
        self.ctx.check(self.ctx._L.hdgb_precond_get(self._h, name.encode(), _ptr(out), n.value, C.byref(n)))
        return out

    @property
    def ritz(self) -> np.ndarray:
        r = self.get("ritz")
        return r[0::2] + 1j * r[1::2]

    def set_ritz(self, theta):
        th = np.asarray(theta, dtype=np.complex128)
        buf = np.empty(2 * len(th))
        buf[0::2], buf[1::2] = th.real, th.imag
        self.ctx.check(self.ctx._L.hdgb_precond_set_ritz(self._h, _ptr(buf), len(th)))

    def apply_base(self, y, z=None):
        """make_base_apply (preconditioner.cpp:285-299)."""
        y = _f64(y)
        out = np.empty(self._n_vec) if z is None else z
        self.ctx.check(self.ctx._L.hdgb_precond_apply_base(self._h, _ptr(y), _ptr(out)))
        return out

    def apply(self, y, z=None):
        """make_preconditioner_apply (preconditioner.cpp:301-308)."""
        y = _f64(y)
        out = np.empty(self._n_vec) if z is None else z
        self.ctx.check(self.ctx._L.hdgb_precond_apply(self._h, self.k._h, _ptr(y), _ptr(out)))
        return out

    @property
    def inner_ops(self) -> int:
        return self.ctx._L.hdgb_precond_inner_ops(self._h)


def build_preconditioner(spec, k: FaceBlockMatrix, ops: ElementOperators = None, disc: Discretization = None) -> Preconditioner:
    """build_preconditioner (newton.cpp:30-52).  spec: PrecondSpec or kind name."""
    if not isinstance(spec, PrecondSpec):
        spec = PrecondSpec(spec)
    h = _vp()
    k.ctx.check(k.ctx._L.hdgb_build_preconditioner(k._h, ops._h if ops else None, disc._h if disc else None,
                                                   C.byref(spec), C.byref(h)))
    return Preconditioner(k.ctx, h, k)


def build_bj(k: FaceBlockMatrix) -> Preconditioner:
    """build_bj (preconditioner.cpp:30-46)."""
    h = _vp()
    k.ctx.check(k.ctx._L.hdgb_build_bj(k._h, C.byref(h)))
    return Preconditioner(k.ctx, h, k)


def build_asm(ops: ElementOperators, disc: Discretization, k: FaceBlockMatrix = None) -> Preconditioner:
    """build_asm (preconditioner.cpp:54-84) from the element operators and the mesh alone; k is only kept for the
    vector size of Preconditioner.apply*."""
    h = _vp()
    disc.ctx.check(disc.ctx._L.hdgb_build_asm(ops._h, disc._h, C.byref(h)))
    return Preconditioner(disc.ctx, h, k if k is not None else disc)


def apply_bj(p: Preconditioner, y, z=None):
    """apply_bj (preconditioner.cpp:48-52)."""
    y = _f64(y)
    out = np.empty(len(y)) if z is None else z
    p.ctx.check(p.ctx._L.hdgb_apply_bj(p._h, _ptr(y), _ptr(out)))
    return out


def apply_asm(p: Preconditioner, y, z=None):
    """apply_asm (preconditioner.cpp:86-105)."""
    y = _f64(y)
    out = np.empty(len(y)) if z is None else z
    p.ctx.check(p.ctx._L.hdgb_apply_asm(p._h, _ptr(y), _ptr(out)))
    return out


def precond_from_host(ctx: Context, kind, mpf, nf, inv=None, disc: Discretization = None, ritz=None, k=None) -> Preconditioner:
    """A Preconditioner from caller data (hdgb_precond_create): the reference's value type handed to the device."""
    kd = PRECONDS[kind] if isinstance(kind, str) else int(kind)
    buf, n = None, 0
    if ritz is not None and len(ritz):
        th = np.asarray(ritz, dtype=np.complex128)
        buf = np.empty(2 * len(th))
        buf[0::2], buf[1::2] = th.real, th.imag
        n = len(th)
    h = _vp()
    inv = _f64(inv)
    ctx.check(ctx._L.hdgb_precond_create(ctx._h, kd, mpf, nf, disc._h if disc else None, _ptr(inv), _ptr(buf), n, C.byref(h)))
    return Preconditioner(ctx, h, k)


def ops_from_host(disc: Discretization, kbar, ebar_inv, fbar, hbar, rbar, ru, ruhat_e=None) -> ElementOperators:
    """ElementOperators from caller data (hdgb_ops_create)."""
    arrs = [_f64(a) for a in (kbar, ebar_inv, fbar, hbar, rbar, ru, ruhat_e)]
    h = _vp()
    disc.ctx.check(disc.ctx._L.hdgb_ops_create(disc._h, *[_ptr(a) for a in arrs], C.byref(h)))
    return ElementOperators(disc, h)


def _wrap_op(fn, errors):
    """Python callable (in_ptr, out_ptr, n) on device addresses -> hdgb_op_fn; exceptions are parked in `errors`."""
    if fn is None:
        return C.cast(None, OP_FN)

    def thunk(_user, din, dout, n):
        try:
            fn(din, dout, n)
            return 0
        except BaseException as e:  # must not propagate through the C frames
            errors.append(e)
            return 1
    return OP_FN(thunk)


def compute_harmonic_ritz(ctx: Context, op, n_dof: int, degree: int, seed: int = 12345) -> np.ndarray:
    """compute_harmonic_ritz (preconditioner.cpp:119-205) of a callable op(in_ptr, out_ptr, n) on device vectors."""
    errors = []
    cb = _wrap_op(op, errors)
    out = np.empty(2 * max(degree, 1))
    n = C.c_int()
    st = ctx._L.hdgb_compute_harmonic_ritz(ctx._h, cb, None, n_dof, degree, seed, _ptr(out), C.byref(n))
    if errors:
        raise errors[0]
    ctx.check(st)
    return out[0:2 * n.value:2] + 1j * out[1:2 * n.value:2]


def apply_poly(p: Preconditioner, k: FaceBlockMatrix, y, base=None, z=None):
    """apply_poly (preconditioner.cpp:246-283); base = callable(in_ptr, out_ptr, n) on device vectors or None (p's own
    base).  Returns (z, inner operator applications)."""
    errors = []
    cb = _wrap_op(base, errors)
    y = _f64(y)
    out = np.empty(k.n_vec) if z is None else z
    ops = C.c_int64(0)
    st = p.ctx._L.hdgb_apply_poly(p._h, cb, None, k._h, _ptr(y), _ptr(out), C.byref(ops))
    if errors:
        raise errors[0]
    p.ctx.check(st)
    return out, ops.value


def gmres_solve_fn(ctx: Context, n: int, matvec, precond, rhs, x0=None, cfg: GmresConfig = None, x=None):
    """gmres_solve (gmres.cpp:61-228), closure form of gmres.hpp:50-53: matvec / precond are callables
    (in_ptr, out_ptr, n) on device vectors (precond None = identity).  Returns (x, GmresStats)."""
    cfg = cfg or GmresConfig()
    errors = []
    mv, pc = _wrap_op(matvec, errors), _wrap_op(precond, errors)
    rhs, x0 = _f64(rhs), _f64(x0)
    out = np.empty(n) if x is None else x
    st = GmresStats()
    trace = np.zeros(max(cfg.max_iters, 1)) if cfg.track_diagnostics else None
    rc = ctx._L.hdgb_gmres_solve_fn(ctx._h, n, mv, None, pc, None, _ptr(rhs), _ptr(x0), C.byref(cfg), _ptr(out), C.byref(st),
                                    _ptr(trace))
    if errors:
        raise errors[0]
    ctx.check(rc)
    if trace is not None:
        st.residual_trace = trace[: st.iters]
    return out, st


def leja_order(theta) -> np.ndarray:
    L = load_library()
    th = np.asarray(theta, dtype=np.complex128)
    buf = np.empty(2 * len(th))
    buf[0::2], buf[1::2] = th.real, th.imag
    out = np.empty(4 * len(th) + 2)
    n = C.c_int()
    st = L.hdgb_leja_order(_ptr(buf), len(th), _ptr(out), C.byref(n))
    if st != 0:
        raise HdgError("leja_order failed")
    return out[0:2 * n.value:2] + 1j * out[1:2 * n.value:2]


def harmonic_ritz_from_hessenberg(hess, pmax, p_eff) -> np.ndarray:
    L = load_library()
    hs = _f64(hess)
    out = np.empty(4 * pmax + 2)
    n = C.c_int()
    st = L.hdgb_harmonic_ritz_from_hessenberg(_ptr(hs), pmax, p_eff, _ptr(out), C.byref(n))
    if st != 0:
        raise HdgError("harmonic_ritz_from_hessenberg failed")
    return out[0:2 * n.value:2] + 1j * out[1:2 * n.value:2]


# ---- Krylov / Newton -------------------------------------------------------------------------------
def gmres_solve(k: FaceBlockMatrix, precond: Preconditioner, rhs, x0=None, cfg: GmresConfig = None, x=None):
    """gmres_solve (gmres.cpp:61-228), data form.  Returns (x, GmresStats)."""
    cfg = cfg or GmresConfig()
    rhs = _f64(rhs)
    x0 = _f64(x0)
    out = np.empty(k.n_vec) if x is None else x
    st = GmresStats()
    trace = np.zeros(cfg.max_iters) if cfg.track_diagnostics else None
    k.ctx.check(k.ctx._L.hdgb_gmres_solve(k._h, precond._h if precond else None, _ptr(rhs), _ptr(x0), C.byref(cfg),
                                          _ptr(out), C.byref(st), _ptr(trace)))
    if trace is not None:
        st.residual_trace = trace[: st.iters]
    return out, st


def orthogonalize(ctx: Context, basis, w, mode="cgs"):
    """orthogonalize (gmres.cpp:28-59) on host arrays: basis (nvec, n), w (n).  Returns (h, w_normalised)."""
    V = _f64(basis).reshape(-1, len(w)) if len(basis) else np.zeros((0, len(w)))
    nvec, n = V.shape
    dV, dw = ctx.alloc(max(V.size, 1)), ctx.alloc(n)
    try:
        if V.size:
            ctx.copy(dV, V, V.size)
        wv = _f64(w).copy()
        ctx.copy(dw, wv, n)
        h = np.empty(nvec + 1)
        ctx.check(ctx._L.hdgb_orthogonalize(ctx._h, dV, nvec, n, dw, 1 if mode == "mgs" else 0, _ptr(h)))
        ctx.copy(wv, dw, n)
    finally:
        ctx.free(dV)
        ctx.free(dw)
    return h, wv


def newton_solve(disc, model, state, ncfg: NewtonConfig = None, gcfg: GmresConfig = None, pspec: PrecondSpec = None,
                 dt=None, u_prev=None) -> SolveReport:
    """newton_solve (newton.cpp:54-154); updates `state` in place."""
    ncfg, gcfg, pspec = ncfg or NewtonConfig(), gcfg or GmresConfig(), pspec or PrecondSpec()
    t, keep = _time(dt, u_prev)
    rep = _Report()
    st = disc.ctx._L.hdgb_newton_solve(disc._h, model._h, state._h, C.byref(ncfg), C.byref(gcfg), C.byref(pspec),
                                       C.byref(t) if t else None, C.byref(rep))
    try:
        disc.ctx.check(st)
    except HdgError as e:
        e.report = SolveReport(rep)
        raise
    return SolveReport(rep)


def time_march(disc, model, state, dt, n_steps, ncfg=None, gcfg=None, pspec=None):
    """time_march (newton.cpp:156-175): n_steps backward-Euler steps."""
    ncfg, gcfg, pspec = ncfg or NewtonConfig(), gcfg or GmresConfig(), pspec or PrecondSpec()
    reps = (_Report * n_steps)()
    disc.ctx.check(disc.ctx._L.hdgb_time_march(disc._h, model._h, state._h, dt, n_steps, C.byref(ncfg), C.byref(gcfg),
                                               C.byref(pspec), reps))
    return [SolveReport(r) for r in reps]
