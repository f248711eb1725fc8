"""Thin ctypes binding of include/de.h (argument marshalling only — every step of the solve
runs in libde's sm_100a kernels).  Function names mirror the C ABI.  There is no CPU path:
if libde.so is missing or no CUDA device is present, the calls fail loudly."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libde.so")

DE_OK, DE_EINVAL, DE_ENOTSPD, DE_ENOCONV, DE_EBREAKDOWN, DE_ESTATE, DE_ENOMEM, DE_ECUDA, DE_ENCCL = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
_NAMES = {0: "DE_OK", -1: "DE_EINVAL", -2: "DE_ENOTSPD", -3: "DE_ENOCONV", -4: "DE_EBREAKDOWN",
          -5: "DE_ESTATE", -6: "DE_ENOMEM", -7: "DE_ECUDA", -8: "DE_ENCCL"}


class DEError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


class de_mesh_t(C.Structure):
    _fields_ = [("dim", C.c_int32), ("nel", C.c_int32 * 3), ("h", C.c_double),
                ("fixed", C.POINTER(C.c_uint8))]


class de_partition_t(C.Structure):
    _fields_ = [("sub", C.c_int32 * 3)]


class de_options_t(C.Structure):
    _fields_ = [("theta", C.c_double), ("lanczos_k", C.c_int32), ("inner_mode", C.c_int32),
                ("inner_tol", C.c_double), ("inner_max_iter", C.c_int32), ("max_iter", C.c_int32),
                ("beta_variant", C.c_int32), ("warm_start", C.c_int32), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("device", C.c_int32), ("nccl_id", C.c_void_p),
                ("stream", C.c_void_p), ("check_every", C.c_int32), ("use_graph", C.c_int32),
                ("host_only", C.c_int32), ("prec_kernels", C.c_int32), ("schur_mode", C.c_int32),
                ("weighted_trace", C.c_int32),
                ("outer", C.c_int32), ("restart", C.c_int32), ("loopback", C.c_void_p)]


class de_stats_t(C.Structure):
    _fields_ = [("ndof", C.c_int64), ("n_free", C.c_int64), ("n_I", C.c_int64), ("n_Gamma", C.c_int64),
                ("n_sub", C.c_int64), ("n_sub_local", C.c_int64), ("band", C.c_int32),
                ("iterations", C.c_int32), ("restarts", C.c_int32), ("relres_recursive", C.c_double),
                ("relres_true", C.c_double), ("ms_factor", C.c_double), ("ms_solve", C.c_double),
                ("ms_pcg", C.c_double), ("ms_schur", C.c_double), ("bytes_factor", C.c_double),
                ("bytes_iter", C.c_double), ("launches_per_iter", C.c_int32),
                ("singular_components", C.c_int32), ("n_cross", C.c_int64 * 3), ("n_faces", C.c_int64 * 3),
                ("n_gamma_c", C.c_int64 * 3),
                ("bytes_schur", C.c_double), ("kernels_launched", C.c_int64),
                ("iterations_pass1", C.c_int32), ("schur_explicit", C.c_int32),
                ("bytes_schur_explicit", C.c_double),
                ("bytes_prec", C.c_double), ("inner_iterations", C.c_int64), ("relres_dd", C.c_double),
                ("bytes_prec_min", C.c_double), ("cross_fd", C.c_int32)]


class de_oc_params_t(C.Structure):
    _fields_ = [("volfrac", C.c_double), ("move", C.c_double), ("rho_min", C.c_double), ("eta", C.c_double),
                ("tol", C.c_double), ("maxit", C.c_int32)]


_lib = None


def lib():
    """Load libde.so (built by __graft_entry__.build() / python -m paper_1501_06211_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libde.so not found at {LIB_PATH}; build it with "
                           "`python -m paper_1501_06211_b200.build` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "de_default_options": (None, [C.POINTER(de_options_t)]),
        "de_setup": (I32, [C.POINTER(de_mesh_t), P, D, D, D, D, C.POINTER(de_partition_t),
                           C.POINTER(de_options_t), C.POINTER(P)]),
        "de_update_densities": (I32, [P, P]),
        "de_update_densities_device": (I32, [P, P]),
        "de_factor": (I32, [P]),
        "de_solve": (I32, [P, P, D, P, C.POINTER(I32), C.POINTER(D)]),
        "de_solve_device": (I32, [P, P, D, P, C.POINTER(I32), C.POINTER(D)]),
        "de_get_dofmap": (I32, [P, P, P, P, C.POINTER(I64), C.POINTER(I64)]),
        "de_get_skeleton": (I32, [P, I32, P, P]),
        "de_get_stats": (I32, [P, C.POINTER(de_stats_t)]),
        "de_get_owned": (I32, [P, P, C.POINTER(I32)]),
        "de_schur_apply_device": (I32, [P, P, P]),
        "de_precond_apply_device": (I32, [P, P, P]),
        "de_get_factor_band": (I32, [P, I32, P, C.POINTER(I32)]),
        "de_get_assembled_band": (I32, [P, I32, P, C.POINTER(I32)]),
        "de_nccl_unique_id": (I32, [P]),
        "de_set_profiling": (I32, [P, I32]),
        "de_get_kernel_time": (I32, [P, C.POINTER(D), C.POINTER(I64)]),
        "de_get_prec_time": (I32, [P, C.POINTER(D), C.POINTER(I64)]),
        "de_default_oc_params": (None, [C.POINTER(de_oc_params_t)]),
        "de_sensitivities_device": (I32, [P, P, P, C.POINTER(D)]),
        "de_oc_update_device": (I32, [P, P, C.POINTER(de_oc_params_t), P, C.POINTER(D)]),
        "de_oc_step": (I32, [P, P, C.POINTER(de_oc_params_t), P, C.POINTER(D), C.POINTER(D)]),
        "de_destroy": (None, [P]),
        "de_last_error": (C.c_char_p, []),
        "de_loopback_create": (I32, [I32, C.POINTER(P)]),
        "de_loopback_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status, allow=()):
    if status != DE_OK and status not in allow:
        raise DEError(status, lib().de_last_error().decode())
    return status


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- C-ABI mirrors

def de_default_options(**kw) -> de_options_t:
    o = de_options_t()
    lib().de_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def de_setup(dim, nel, h, fixed, density, E0, Emin, p, nu, sub, options=None):
    fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
    density = np.ascontiguousarray(density, dtype=np.float64)
    m = de_mesh_t()
    m.dim = dim
    for a in range(3):
        m.nel[a] = int(nel[a]) if a < dim else 1
    m.h = float(h)
    m.fixed = fixed.ctypes.data_as(C.POINTER(C.c_uint8))
    part = de_partition_t()
    for a in range(3):
        part.sub[a] = int(sub[a]) if a < dim else 1
    opt = options if options is not None else de_default_options()
    ctx = C.c_void_p()
    _check(lib().de_setup(C.byref(m), _ptr(density), E0, Emin, p, nu, C.byref(part), C.byref(opt),
                          C.byref(ctx)))
    return ctx


def de_update_densities(ctx, density):
    density = np.ascontiguousarray(density, dtype=np.float64)
    _check(lib().de_update_densities(ctx, _ptr(density)))


def de_update_densities_device(ctx, d_density_ptr: int):
    _check(lib().de_update_densities_device(ctx, C.c_void_p(d_density_ptr)))


def de_factor(ctx):
    _check(lib().de_factor(ctx))


def de_solve(ctx, rhs, rtol, u=None, allow_noconv=False):
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    u = np.empty_like(rhs) if u is None else u
    it, rr = C.c_int32(), C.c_double()
    st = _check(lib().de_solve(ctx, _ptr(rhs), rtol, _ptr(u), C.byref(it), C.byref(rr)),
                allow=(DE_ENOCONV,) if allow_noconv else ())
    return u, it.value, rr.value, st


def de_solve_device(ctx, d_rhs_ptr: int, rtol, d_u_ptr: int, allow_noconv=False):
    it, rr = C.c_int32(), C.c_double()
    st = _check(lib().de_solve_device(ctx, C.c_void_p(d_rhs_ptr), rtol, C.c_void_p(d_u_ptr),
                                      C.byref(it), C.byref(rr)),
                allow=(DE_ENOCONV,) if allow_noconv else ())
    return it.value, rr.value, st


def de_get_stats(ctx) -> de_stats_t:
    s = de_stats_t()
    _check(lib().de_get_stats(ctx, C.byref(s)))
    return s


def de_get_owned(ctx):
    n = C.c_int32()
    _check(lib().de_get_owned(ctx, None, C.byref(n)))
    ids = np.empty(n.value, np.int32)
    _check(lib().de_get_owned(ctx, _ptr(ids), C.byref(n)))
    return ids


def de_get_dofmap(ctx):
    s = de_get_stats(ctx)
    n = s.ndof
    cls = np.empty(n, np.int8)
    sub = np.empty(n, np.int32)
    red = np.empty(n, np.int32)
    nI, nG = C.c_int64(), C.c_int64()
    _check(lib().de_get_dofmap(ctx, _ptr(cls), _ptr(sub), _ptr(red), C.byref(nI), C.byref(nG)))
    return cls, sub, red, nI.value, nG.value


def de_get_skeleton(ctx, c):
    s = de_get_stats(ctx)
    n = s.n_gamma_c[c]
    nodes = np.empty(n, np.int32)
    face = np.empty(n, np.int32)
    _check(lib().de_get_skeleton(ctx, c, _ptr(nodes), _ptr(face)))
    return nodes, face


def de_schur_apply_device(ctx, d_p_ptr: int, d_q_ptr: int):
    _check(lib().de_schur_apply_device(ctx, C.c_void_p(d_p_ptr), C.c_void_p(d_q_ptr)))


def de_precond_apply_device(ctx, d_r_ptr: int, d_z_ptr: int):
    _check(lib().de_precond_apply_device(ctx, C.c_void_p(d_r_ptr), C.c_void_p(d_z_ptr)))


def _band(fn, ctx, sl):
    s = de_get_stats(ctx)
    n = C.c_int32()
    _check(fn(ctx, sl, None, C.byref(n)))
    out = np.empty((n.value, s.band + 1))
    _check(fn(ctx, sl, _ptr(out), C.byref(n)))
    return out


def de_get_factor_band(ctx, sl):
    return _band(lib().de_get_factor_band, ctx, sl)


def de_get_assembled_band(ctx, sl):
    return _band(lib().de_get_assembled_band, ctx, sl)


def de_nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().de_nccl_unique_id(buf))
    return bytes(buf)


def de_set_profiling(ctx, on: bool):
    _check(lib().de_set_profiling(ctx, 1 if on else 0))


def de_get_kernel_time(ctx):
    ms, n = C.c_double(), C.c_int64()
    _check(lib().de_get_kernel_time(ctx, C.byref(ms), C.byref(n)))
    return ms.value, n.value


def de_get_prec_time(ctx):
    ms, n = C.c_double(), C.c_int64()
    _check(lib().de_get_prec_time(ctx, C.byref(ms), C.byref(n)))
    return ms.value, n.value


def de_default_oc_params(**kw) -> de_oc_params_t:
    o = de_oc_params_t()
    lib().de_default_oc_params(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def de_sensitivities_device(ctx, d_u_ptr: int, d_dc_ptr: int | None = None, want_compliance=True):
    c = C.c_double()
    _check(lib().de_sensitivities_device(ctx, C.c_void_p(d_u_ptr), C.c_void_p(d_dc_ptr) if d_dc_ptr else None,
                                         C.byref(c) if want_compliance else None))
    return c.value if want_compliance else None


def de_oc_update_device(ctx, d_dc_ptr: int | None, params: de_oc_params_t, d_rho_new_ptr: int | None = None):
    lam = C.c_double()
    _check(lib().de_oc_update_device(ctx, C.c_void_p(d_dc_ptr) if d_dc_ptr else None, C.byref(params),
                                     C.c_void_p(d_rho_new_ptr) if d_rho_new_ptr else None, C.byref(lam)))
    return lam.value


def de_oc_step(ctx, u, params: de_oc_params_t, nelem: int):
    u = np.ascontiguousarray(u, dtype=np.float64)
    rho = np.empty(nelem, np.float64)
    c, lam = C.c_double(), C.c_double()
    _check(lib().de_oc_step(ctx, _ptr(u), C.byref(params), _ptr(rho), C.byref(c), C.byref(lam)))
    return rho, c.value, lam.value


def de_loopback_create(nranks: int):
    g = C.c_void_p()
    _check(lib().de_loopback_create(int(nranks), C.byref(g)))
    return g


def de_loopback_destroy(g):
    if g:
        lib().de_loopback_destroy(g)


def de_destroy(ctx):
    if ctx:
        lib().de_destroy(ctx)


# ----------------------------------------------------------------- convenience wrapper

class Solver:
    """RAII wrapper: Solver(problem-like, **options) -> factor() -> solve(rhs)."""

    def __init__(self, dim, nel, sub, fixed, density, E0=1.0, Emin=1e-9, p=3.0, nu=0.3, h=1.0,
                 nccl_id: bytes | None = None, **opts):
        self._idbuf = None
        if nccl_id is not None:
            self._idbuf = C.create_string_buffer(nccl_id, 128)
            opts["nccl_id"] = C.cast(self._idbuf, C.c_void_p)
        self.options = de_default_options(**opts)
        self.ctx = de_setup(dim, nel, h, fixed, density, E0, Emin, p, nu, sub, self.options)

    @classmethod
    def from_problem(cls, prob, **opts):
        return cls(prob.dim, prob.nel, prob.sub, prob.fixed, prob.density, prob.E0, prob.Emin, prob.p,
                   prob.nu, prob.h, **opts)

    def factor(self):
        de_factor(self.ctx)

    def update_densities(self, rho):
        de_update_densities(self.ctx, rho)

    def solve(self, rhs, rtol=1e-10, allow_noconv=False):
        return de_solve(self.ctx, rhs, rtol, allow_noconv=allow_noconv)

    def oc_step(self, u, nelem, **params):
        """One optimality-criteria design update from the displacement u (R20); the new densities
        replace the context's, so factor() must be called before the next solve."""
        return de_oc_step(self.ctx, u, de_default_oc_params(**params), nelem)

    def stats(self):
        return de_get_stats(self.ctx)

    def dofmap(self):
        return de_get_dofmap(self.ctx)

    def close(self):
        if self.ctx:
            de_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
