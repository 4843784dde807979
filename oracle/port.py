"""TEST INFRASTRUCTURE ONLY: ctypes wrapper over oracle/libhdgoracle.so (hdg_oracle.cpp), the
generalised CPU restatement of the reference hot path (2D/3D, M components).  Used by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm; never by the product.

The restatement takes the discretisation TABLES as input.  tests/test_oracle.py pins it bit for bit
against the unmodified reference (oracle/_ref) with the reference's own tables on 2D quads."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libhdgoracle.so"
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lib = None

MODELS = {"poisson": 0, "burgers": 1, "convdiff": 2, "elasticity": 3, "reaction": 4, "navier_stokes": 5}
PRECOND = {"none": 0, "identity": 0, "bj": 1, "asm": 2, "ras": 3}
POLY = {"gmres": 0, "chebyshev": 1}


class OracleError(RuntimeError):
    def __init__(self, code, msg, index=-1):
        super().__init__(f"[{code}] {msg}")
        self.code, self.index = code, index


def build():
    subprocess.check_call(["make", "-s", "-C", str(_HERE), "oracle"])


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.ora_create.restype = C.c_void_p
        L.ora_create.argtypes = [_ip] * 7 + [_dp] * 14
        L.ora_free.argtypes = [C.c_void_p]
        L.ora_last_error.restype = C.c_char_p
        L.ora_last_error.argtypes = [C.c_void_p]
        L.ora_last_error_index.restype = C.c_long
        L.ora_last_error_index.argtypes = [C.c_void_p]
        L.ora_set_model.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, _dp, _dp]
        L.ora_local_factors.argtypes = [C.c_void_p]
        L.ora_get.restype = C.c_long
        L.ora_get.argtypes = [C.c_void_p, C.c_char_p, _dp, C.c_long]
        L.ora_set.argtypes = [C.c_void_p, C.c_char_p, _dp, C.c_long]
        L.ora_get_neighbor.restype = C.c_long
        L.ora_get_neighbor.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_long]
        L.ora_get_gmres_per_newton.restype = C.c_long
        L.ora_get_gmres_per_newton.argtypes = [C.c_void_p, _ip, C.c_long]
        L.ora_set_dt.argtypes = [C.c_void_p, C.c_double]
        L.ora_compute_q.argtypes = [C.c_void_p]
        L.ora_assemble_core.argtypes = [C.c_void_p, C.c_int]
        L.ora_assemble_element_operators.argtypes = [C.c_void_p]
        L.ora_assemble_global.argtypes = [C.c_void_p]
        L.ora_matvec.argtypes = [C.c_void_p, _dp, _dp]
        L.ora_build_precond.argtypes = [C.c_void_p, C.c_int]
        L.ora_apply_base.argtypes = [C.c_void_p, _dp, _dp]
        L.ora_apply_precond.argtypes = [C.c_void_p, _dp, _dp]
        L.ora_residual.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ora_recover_local.argtypes = [C.c_void_p, _dp, _dp]
        L.ora_gmres.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ora_newton.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.c_int, C.c_uint64, _dp]
        L.ora_build_poly.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64]
        L.ora_set_threads.argtypes = [C.c_int]
        L.ora_lu_invert_batch.argtypes = [C.c_int, C.c_int, _dp, _dp, C.POINTER(C.c_long)]
        _lib = L
    return _lib


def set_threads(n: int):
    lib().ora_set_threads(int(n))


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _pi(a):
    return a.ctypes.data_as(_ip)


def tables_from_disc(disc) -> dict:
    """Discretisation tables from the product's host-side setup layer (paper_2512_13619_b200
    Discretization.table); on 2D quads these are checked bit for bit against the reference."""
    t = dict(D=disc.dim, M=disc.n_comp, ne=disc.ne, nf=disc.nf, n_lfe=disc.n_lfe, n_orient=disc.n_orient,
             pe=disc.pe, pf=disc.pf, qe=disc.qe, qf=disc.qf)
    t["elem_faces"] = disc.table("element_to_face")
    t["elem_side"] = disc.table("elem_side")
    t["face_elems"] = disc.table("face_to_elements")
    t["face_lidx"] = disc.table("face_local_index")
    t["face_orient"] = disc.table("face_orient")
    t["bnd_tag"] = disc.table("boundary_tag")
    for k in ("phi", "dphi0", "dphi1", "psi", "tphi", "elem_detjac", "elem_invjac", "elem_coords", "face_detjac",
              "face_coords", "face_normal"):
        t[k] = disc.table(k)
    t["dphi2"] = disc.table("dphi2") if disc.dim == 3 else None
    t["wq"], t["wf"] = disc.table("elem_weights"), disc.table("face_weights")
    return t


def tables_from_ref(rc, n_comp=1) -> dict:
    """The REFERENCE's own tables (oracle/_ref RefCase) in this oracle's layout."""
    ne, nf, pe, pf, qe, qf = rc.ne, rc.nf, rc.pe, rc.pf, rc.qe, rc.qf
    e2f = rc.get_i("element_to_face").reshape(ne, 4)
    f2e = rc.get_i("face_to_elements").reshape(nf, 2)
    fli = rc.get_i("face_local_index").reshape(nf, 2)
    rev = rc.get_i("face_side_reversed").reshape(nf, 2)
    side = np.zeros((ne, 4), dtype=np.int32)
    for e in range(ne):
        for lf in range(4):
            f = e2f[e, lf]
            side[e, lf] = 0 if (f2e[f, 0] == e and fli[f, 0] == lf) else 1   # local_ops.cpp:129-132
    tl = np.stack([rc.get(f"trace_phi{l}").reshape(qf, pe) for l in range(4)])  # [lf][g][i]
    tphi = np.stack([tl, tl[:, ::-1, :]], axis=1)                              # [lf][o][gc][i], gs = qf-1-gc
    t = dict(D=2, M=n_comp, ne=ne, nf=nf, n_lfe=4, n_orient=2, pe=pe, pf=pf, qe=qe, qf=qf,
             elem_faces=e2f, elem_side=side, face_elems=f2e, face_lidx=fli, face_orient=rev,
             bnd_tag=rc.get_i("boundary_tag"), phi=rc.get("phi"), dphi0=rc.get("dphi_dxi"), dphi1=rc.get("dphi_deta"),
             dphi2=None, psi=rc.get("psi"), tphi=tphi, wq=rc.get("rule2d_weights"), wf=rc.get("rule1d_weights"))
    for k in ("elem_detjac", "elem_invjac", "elem_coords", "face_detjac", "face_coords", "face_normal"):
        t[k] = rc.get(k)
    return t


class OraCase:
    def __init__(self, t: dict):
        L = lib()
        self.t = t
        for k in ("D", "M", "ne", "nf", "n_lfe", "n_orient", "pe", "pf", "qe", "qf"):
            setattr(self, k, int(t[k]))
        self.npe, self.mpf = self.M * self.pe, self.M * self.pf
        self.nfl, self.nb, self.n_dof = self.n_lfe * self.mpf, 2 * self.n_lfe - 1, self.mpf * self.nf
        dims = _i([self.D, self.M, self.ne, self.nf, self.n_lfe, self.n_orient, self.pe, self.pf, self.qe, self.qf])
        ints = [_i(t[k]) for k in ("elem_faces", "elem_side", "face_elems", "face_lidx", "face_orient", "bnd_tag")]
        dbl = [_d(t[k]) for k in ("phi", "dphi0", "dphi1", "dphi2", "psi", "tphi", "wq", "wf", "elem_detjac",
                                  "elem_invjac", "elem_coords", "face_detjac", "face_coords", "face_normal")]
        self._h = L.ora_create(_pi(dims), *[_pi(a) for a in ints], *[_p(a) for a in dbl])
        self._check(L.ora_local_factors(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ora_free(self._h)
            self._h = None

    def _check(self, rc):
        if rc != 0:
            L = lib()
            raise OracleError(rc, L.ora_last_error(self._h).decode(), L.ora_last_error_index(self._h))

    def set_model(self, kind: str, params, forcing_q=None, dirichlet_q=None):
        p = _d(params)
        f, g = _d(forcing_q), _d(dirichlet_q)
        lib().ora_set_model(self._h, MODELS[kind], _p(p), len(p), _p(f), _p(g))

    def set_model_like(self, model):
        """Same functor tag / parameters / tabulated data as a product Model (hdg.Model)."""
        disc = model.disc
        fq = dq = None
        # re-tabulate from the Python callbacks kept on the model (same numpy expressions)
        if getattr(model, "_forcing", None) is not None or getattr(model, "_dirichlet", None) is not None:
            xq, xf = disc.quad_coords()
            if model._forcing is not None:
                fq = np.broadcast_to(np.asarray(model._forcing(xq), dtype=np.float64).reshape(disc.ne, disc.qe, -1),
                                     (disc.ne, disc.qe, disc.n_comp))
            if model._dirichlet is not None:
                dq = np.broadcast_to(np.asarray(model._dirichlet(xf), dtype=np.float64).reshape(disc.nf, disc.qf, -1),
                                     (disc.nf, disc.qf, disc.n_comp))
        self.set_model(model.kind, model.params, fq, dq)

    def get(self, name):
        L = lib()
        n = L.ora_get(self._h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n)
        L.ora_get(self._h, name.encode(), _p(out), n)
        return out

    def set(self, name, v):
        v = _d(v)
        if lib().ora_set(self._h, name.encode(), _p(v), v.size) != 0:
            raise KeyError(name)

    @property
    def neighbor(self):
        L = lib()
        n = L.ora_get_neighbor(self._h, None, 0)
        out = np.empty(n, dtype=np.int64)
        L.ora_get_neighbor(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)), n)
        return out

    def set_dt(self, dt, u_prev=None):
        lib().ora_set_dt(self._h, -1.0 if dt is None else float(dt))
        if u_prev is not None:
            self.set("u_prev", u_prev)

    def compute_q(self):
        lib().ora_compute_q(self._h)

    def assemble_core(self, want_jac=True):
        self._check(lib().ora_assemble_core(self._h, int(want_jac)))

    def assemble(self):
        self._check(lib().ora_assemble_element_operators(self._h))
        lib().ora_assemble_global(self._h)

    def matvec(self, x):
        x = _d(x)
        y = np.empty_like(x)
        lib().ora_matvec(self._h, _p(x), _p(y))
        return y

    def build_precond(self, kind="bj", poly_degree=0, poly_kind="gmres", seed=12345):
        """build_bj / build_asm (+ RAS) and, for poly_degree > 0, the harmonic-Ritz (or Chebyshev) nodes."""
        self._check(lib().ora_build_precond(self._h, PRECOND[kind]))
        if poly_degree > 0:
            self._check(lib().ora_build_poly(self._h, poly_degree, POLY[poly_kind], seed))

    @property
    def ritz(self):
        r = self.get("ritz")
        return r[0::2] + 1j * r[1::2]

    def set_ritz(self, theta):
        th = np.asarray(theta, dtype=np.complex128)
        buf = np.empty(2 * len(th))
        buf[0::2], buf[1::2] = th.real, th.imag
        self.set("ritz", buf)

    def apply_base(self, y):
        y = _d(y)
        z = np.empty_like(y)
        lib().ora_apply_base(self._h, _p(y), _p(z))
        return z

    def apply_precond(self, y):
        y = _d(y)
        z = np.empty_like(y)
        lib().ora_apply_precond(self._h, _p(y), _p(z))
        return z

    def residual(self):
        tr, it = np.empty(self.n_dof), np.empty(self.npe * self.ne)
        nrm = C.c_double()
        self._check(lib().ora_residual(self._h, _p(tr), _p(it), C.byref(nrm)))
        return tr, it, nrm.value

    def recover_local(self, duhat):
        d = _d(duhat)
        du = np.empty(self.npe * self.ne)
        lib().ora_recover_local(self._h, _p(d), _p(du))
        return du

    def gmres(self, rhs=None, x0=None, restart=50, tol=1e-6, max_iters=1000, mgs=False):
        x = np.empty(self.n_dof)
        st = np.zeros(7)
        r, xv = _d(rhs), _d(x0)
        self._check(lib().ora_gmres(self._h, _p(r), _p(xv), restart, tol, max_iters, int(mgs), _p(x), _p(st)))
        return x, dict(iters=int(st[0]), restarts=int(st[1]), final_rel_residual=st[2], converged=bool(st[3]),
                       t_mv=st[4], t_prec=st[5], t_orth=st[6])

    def newton(self, newton_tol=1e-8, max_newton=50, min_alpha=1.0 / 1024.0, restart=50, gmres_tol=1e-6,
               gmres_max_iters=1000, mgs=False, precond="bj", poly_degree=0, poly_kind="gmres", seed=12345,
               dt=None, u_prev=None):
        if dt is not None:
            self.set_dt(dt, u_prev)
        rep = np.zeros(10)
        self._check(lib().ora_newton(self._h, newton_tol, max_newton, min_alpha, restart, gmres_tol, gmres_max_iters,
                                     int(mgs), PRECOND[precond], poly_degree, POLY[poly_kind], seed, _p(rep)))
        keys = ["n_newton", "n_gmres_total", "n_inner_prec_ops", "final_residual", "converged", "t_ass", "t_mv",
                "t_prec", "t_orth", "t_total"]
        d = dict(zip(keys, rep))
        for k in keys[:3]:
            d[k] = int(d[k])
        d["converged"] = bool(d["converged"])
        d["residual_history"] = self.get("residual_history")
        d["alpha_history"] = self.get("alpha_history")
        L = lib()
        n = L.ora_get_gmres_per_newton(self._h, None, 0)
        g = np.zeros(n, dtype=np.int32)
        L.ora_get_gmres_per_newton(self._h, _pi(g), n)
        d["gmres_per_newton"] = g
        return d
