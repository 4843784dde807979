"""TEST INFRASTRUCTURE ONLY: ctypes wrapper over oracle/_ref/libhdgref.so, i.e. the UNMODIFIED
reference (/root/reference/proj) compiled in place by oracle/Makefile.

Used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm as
the checker / timed CPU baseline. The product (paper_2512_13619_b200/) never imports this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_ref" / "libhdgref.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


class RefError(RuntimeError):
    def __init__(self, kind: str, msg: str, index: int):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.index = index


def available() -> bool:
    return LIB_PATH.exists()


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(str(LIB_PATH))
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error_kind.restype = C.c_char_p
        L.ref_last_error_index.restype = C.c_long
        L.ref_case_create.restype = C.c_void_p
        L.ref_case_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_int]
        L.ref_case_free.argtypes = [C.c_void_p]
        L.ref_case_get.restype = C.c_long
        L.ref_case_get.argtypes = [C.c_void_p, C.c_char_p, _dp, C.c_long]
        L.ref_case_get_i.restype = C.c_long
        L.ref_case_get_i.argtypes = [C.c_void_p, C.c_char_p, _ip, C.c_long]
        L.ref_case_set.argtypes = [C.c_void_p, C.c_char_p, _dp, C.c_long]
        L.ref_case_dims.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.ref_case_perturb.argtypes = [C.c_void_p, C.c_uint64, C.c_double]
        L.ref_case_set_dt.argtypes = [C.c_void_p, C.c_double]
        L.ref_case_reset_state.argtypes = [C.c_void_p]
        L.ref_case_compute_q.argtypes = [C.c_void_p]
        L.ref_case_assemble.argtypes = [C.c_void_p, C.c_int]
        L.ref_case_assemble_local.argtypes = [C.c_void_p]
        L.ref_case_assemble_global.argtypes = [C.c_void_p]
        L.ref_case_residual.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_case_matvec.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_case_to_dense.restype = C.c_long
        L.ref_case_to_dense.argtypes = [C.c_void_p, _dp, C.c_long]
        L.ref_case_gather_extended.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_case_build_precond.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64]
        L.ref_case_apply_base.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_case_apply_precond.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_case_set_ritz.argtypes = [C.c_void_p, _dp, C.c_int]
        L.ref_case_gather_element_trace.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_case_recover_local.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_case_gmres.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ref_case_newton.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, _dp]
        L.ref_case_time_march.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                                          C.c_double, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_case_monolithic.restype = C.c_long
        L.ref_case_monolithic.argtypes = [C.c_void_p, _dp, _dp, C.c_long]
        L.ref_case_write_matrix.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_case_l2_error.restype = C.c_double
        L.ref_case_l2_error.argtypes = [C.c_void_p]
        L.ref_lu_invert_batch.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.ref_gemm_batch.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.ref_gemv_strided_batch.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int]
        L.ref_random_vector.argtypes = [C.c_long, C.c_uint64, C.c_double, _dp]
        L.ref_gauss_rule.argtypes = [C.c_int, _dp, _dp]
        L.ref_lobatto_nodes.argtypes = [C.c_int, _dp]
        L.ref_leja_order.argtypes = [C.c_int, _dp, _dp]
        L.ref_harmonic_ritz_dense.argtypes = [C.c_int, _dp, C.c_int, C.c_uint64, _dp]
        L.ref_gmres_dense.argtypes = [C.c_int, _dp, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ref_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(rc):
    if rc != 0:
        L = lib()
        raise RefError(L.ref_last_error_kind().decode(), L.ref_last_error().decode(), L.ref_last_error_index())


def set_threads(n: int):
    lib().ref_set_threads(int(n))


def random_vector(n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty(n)
    lib().ref_random_vector(n, seed, scale, _p(out))
    return out


def lu_invert_batch(a: np.ndarray) -> np.ndarray:
    """a: (batch, n, n) with each block stored column-major => pass arrays shaped (batch, n*n)."""
    a = _f64(a)
    batch = a.shape[0]
    n = int(round(np.sqrt(a.size // batch)))
    out = np.empty_like(a)
    _check(lib().ref_lu_invert_batch(n, batch, _p(a), _p(out)))
    return out


def gemm_batch(a, ar, ac, abatch, b, br, bc, bbatch, transpose_a=False):
    a, b = _f64(a), _f64(b)
    m = ac if transpose_a else ar
    out = np.empty(max(abatch, bbatch) * m * bc)
    _check(lib().ref_gemm_batch(ar, ac, abatch, _p(a), br, bc, bbatch, _p(b), int(transpose_a), _p(out)))
    return out


def gemv_strided_batch(a, rows, cols, batch, x, y=None, accumulate=False):
    a, x = _f64(a), _f64(x)
    yv = np.zeros(rows * batch) if y is None else _f64(y).copy()
    _check(lib().ref_gemv_strided_batch(rows, cols, batch, _p(a), _p(x), _p(yv), int(accumulate)))
    return yv


def gauss_rule(q):
    p, w = np.empty(q), np.empty(q)
    _check(lib().ref_gauss_rule(q, _p(p), _p(w)))
    return p, w


def lobatto_nodes(n):
    out = np.empty(n)
    _check(lib().ref_lobatto_nodes(n, _p(out)))
    return out


def leja_order(theta) -> np.ndarray:
    th = np.asarray(theta, dtype=np.complex128)
    inp = np.empty(2 * len(th))
    inp[0::2], inp[1::2] = th.real, th.imag
    out = np.empty(4 * len(th) + 2)
    n = lib().ref_leja_order(len(th), _p(inp), _p(out))
    return out[0:2 * n:2] + 1j * out[1:2 * n:2]


def harmonic_ritz_dense(a: np.ndarray, degree: int, seed: int) -> np.ndarray:
    a = _f64(a)
    n = a.shape[0]
    out = np.empty(4 * degree + 2)
    cnt = lib().ref_harmonic_ritz_dense(n, _p(a), degree, seed, _p(out))
    if cnt < 0:
        _check(1)
    return out[0:2 * cnt:2] + 1j * out[1:2 * cnt:2]


def gmres_dense(a, rhs, pinv=None, x0=None, restart=50, tol=1e-6, max_iters=1000, mgs=False):
    a, rhs = _f64(a), _f64(rhs)
    n = len(rhs)
    x = np.empty(n)
    st = np.zeros(4)
    pv = _f64(pinv) if pinv is not None else None
    xv = _f64(x0) if x0 is not None else None
    _check(lib().ref_gmres_dense(n, _p(a), _p(pv) if pv is not None else None, _p(rhs),
                                 _p(xv) if xv is not None else None, restart, tol, max_iters, int(mgs),
                                 _p(x), _p(st)))
    return x, dict(iters=int(st[0]), restarts=int(st[1]), final_rel_residual=st[2], converged=bool(st[3]))


PRECOND = {"none": 0, "identity": 0, "bj": 1, "asm": 2}


class RefCase:
    """One reference case (study.cpp:67-77 make_case_setup + make_initial_state)."""

    def __init__(self, case="poisson2d", k=2, n=8, tau=None, nu=1.0 / 200.0, kappa=1.0,
                 velocity=(0.0, 1.0), quad_points=0):
        L = lib()
        self._h = L.ref_case_create(case.encode(), k, n, float("nan") if tau is None else float(tau),
                                    nu, kappa, velocity[0], velocity[1], quad_points)
        if not self._h:
            _check(1)
        d = (C.c_int * 6)()
        L.ref_case_dims(self._h, d)
        self.ne, self.nf, self.pe, self.pf, self.qe, self.qf = list(d)
        self.case, self.k, self.n = case, k, n
        self.n_dof = self.nf * self.pf

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_case_free(self._h)
            self._h = None

    def get(self, name: str) -> np.ndarray:
        L = lib()
        n = L.ref_case_get(self._h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n)
        L.ref_case_get(self._h, name.encode(), _p(out), n)
        return out

    def get_i(self, name: str) -> np.ndarray:
        L = lib()
        n = L.ref_case_get_i(self._h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, dtype=np.int64)
        L.ref_case_get_i(self._h, name.encode(), out.ctypes.data_as(_ip), n)
        return out

    def set(self, name: str, v):
        v = _f64(v)
        rc = lib().ref_case_set(self._h, name.encode(), _p(v), v.size)
        if rc != 0:
            raise ValueError(f"set {name}: rc={rc}")

    def set_dt(self, dt):
        lib().ref_case_set_dt(self._h, -1.0 if dt is None else float(dt))

    def reset_state(self):
        lib().ref_case_reset_state(self._h)

    def perturb(self, seed: int, scale: float):
        lib().ref_case_perturb(self._h, seed, scale)

    def compute_q(self):
        _check(lib().ref_case_compute_q(self._h))

    def assemble(self, keep_raw=False):
        _check(lib().ref_case_assemble(self._h, int(keep_raw)))

    def assemble_local(self):
        _check(lib().ref_case_assemble_local(self._h))

    def assemble_global(self):
        _check(lib().ref_case_assemble_global(self._h))

    def residual(self):
        tr, it = np.empty(self.nf * self.pf), np.empty(self.ne * self.pe)
        nrm = C.c_double()
        _check(lib().ref_case_residual(self._h, _p(tr), _p(it), C.byref(nrm)))
        return tr, it, nrm.value

    def matvec(self, x):
        x = _f64(x)
        y = np.empty_like(x)
        _check(lib().ref_case_matvec(self._h, _p(x), _p(y)))
        return y

    def to_dense(self):
        n = self.n_dof
        out = np.empty(n * n)
        if lib().ref_case_to_dense(self._h, _p(out), out.size) < 0:
            _check(1)
        return out.reshape(n, n)

    def gather_extended(self, x, nb=7):
        x = _f64(x)
        out = np.empty(x.size * nb)
        _check(lib().ref_case_gather_extended(self._h, _p(x), _p(out)))
        return out

    def build_precond(self, kind="bj", poly_degree=0, seed=12345):
        _check(lib().ref_case_build_precond(self._h, PRECOND[kind], poly_degree, seed))

    def set_ritz(self, theta):
        th = np.asarray(theta, dtype=np.complex128)
        buf = np.empty(2 * len(th))
        buf[0::2], buf[1::2] = th.real, th.imag
        _check(lib().ref_case_set_ritz(self._h, _p(buf), len(th)))

    def apply_base(self, y):
        y = _f64(y)
        z = np.empty_like(y)
        _check(lib().ref_case_apply_base(self._h, _p(y), _p(z)))
        return z

    def apply_precond(self, y):
        y = _f64(y)
        z = np.empty_like(y)
        _check(lib().ref_case_apply_precond(self._h, _p(y), _p(z)))
        return z

    def gather_element_trace(self, v):
        v = _f64(v)
        out = np.empty(self.ne * 4 * self.pf)
        _check(lib().ref_case_gather_element_trace(self._h, _p(v), _p(out)))
        return out

    def recover_local(self, duhat):
        duhat = _f64(duhat)
        du = np.empty(self.ne * self.pe)
        _check(lib().ref_case_recover_local(self._h, _p(duhat), _p(du)))
        return du

    def gmres(self, rhs=None, x0=None, restart=50, tol=1e-6, max_iters=1000, mgs=False):
        x = np.empty(self.n_dof)
        st = np.zeros(7)
        r = _f64(rhs) if rhs is not None else None
        xv = _f64(x0) if x0 is not None else None
        _check(lib().ref_case_gmres(self._h, _p(r) if r is not None else None,
                                    _p(xv) if xv is not None else None, restart, tol, max_iters, int(mgs),
                                    _p(x), _p(st)))
        return x, dict(iters=int(st[0]), restarts=int(st[1]), final_rel_residual=st[2], converged=bool(st[3]),
                       t_mv=st[4], t_prec=st[5], t_orth=st[6])

    _REPORT = ["n_newton", "n_gmres_total", "n_inner_prec_ops", "final_residual", "converged",
               "t_ass", "t_mv", "t_prec", "t_orth", "t_total"]

    def _report(self, rep):
        d = dict(zip(self._REPORT, rep))
        for k in ("n_newton", "n_gmres_total", "n_inner_prec_ops"):
            d[k] = int(d[k])
        d["converged"] = bool(d["converged"])
        return d

    def newton(self, newton_tol=1e-8, max_newton=50, min_alpha=1.0 / 1024.0, restart=50, gmres_tol=1e-6,
               gmres_max_iters=1000, mgs=False, precond="bj", poly_degree=0, seed=12345,
               ritz_per_restart=False):
        rep = np.zeros(10)
        _check(lib().ref_case_newton(self._h, newton_tol, max_newton, min_alpha, restart, gmres_tol,
                                     gmres_max_iters, int(mgs), PRECOND[precond], poly_degree, seed,
                                     int(ritz_per_restart), _p(rep)))
        d = self._report(rep)
        d["residual_history"] = self.get("residual_history")
        d["alpha_history"] = self.get("alpha_history")
        d["gmres_per_newton"] = self.get_i("gmres_per_newton")
        return d

    def time_march(self, dt, n_steps, newton_tol=1e-8, max_newton=50, restart=50, gmres_tol=1e-6,
                   gmres_max_iters=1000, precond="bj", poly_degree=0):
        rep = np.zeros(10)
        _check(lib().ref_case_time_march(self._h, dt, n_steps, newton_tol, max_newton, restart, gmres_tol,
                                         gmres_max_iters, PRECOND[precond], poly_degree, _p(rep)))
        return self._report(rep)

    def monolithic(self):
        n = lib().ref_case_monolithic(self._h, None, None, 0)
        if n < 0:
            _check(1)
        a, rhs = np.empty(n * n), np.empty(n)
        lib().ref_case_monolithic(self._h, _p(a), _p(rhs), n)
        return a.reshape(n, n), rhs

    def write_matrix(self, path):
        _check(lib().ref_case_write_matrix(self._h, os.fsencode(path)))

    def l2_error(self):
        return lib().ref_case_l2_error(self._h)
