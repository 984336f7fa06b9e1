"""Thin ctypes binding of libfraccontrol.so (include/fraccontrol.h) — argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only allocates device
buffers with PyTorch, fills the ABI structs and checks status codes.  There is no CPU
fallback: if the shared library is missing, `Library()` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfraccontrol.so")

FC_F, FC_G, FC_POW_PLUS, FC_POW_MINUS = 0, 1, 2, 3
FC_PRECOND_B, FC_PRECOND_A = 0, 1
FC_KP_DOT_REDUCE, FC_KP_KR_BASIS, FC_KP_KR_PRODUCT = 0, 1, 2
FC_MAX_ITERS = 256
STATUS = {0: "OK", 1: "NOT_CONVERGED", 2: "RANK_CAP_HIT", -1: "INVALID_ARG", -2: "SHAPE",
          -3: "CAPACITY", -4: "NONPOS_COEF", -5: "NOT_SPD", -6: "NAN", -7: "EIG_NOCONV",
          -8: "CUDA", -9: "NOT_READY"}


class fc_cp(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("rank", C.c_int), ("cap", C.c_int), ("w", C.c_void_p),
                ("U", C.c_void_p * 3), ("ld", C.c_int * 3)]


class fc_lr2(C.Structure):
    _fields_ = [("n", C.c_int * 2), ("rank", C.c_int), ("cap", C.c_int), ("w", C.c_void_p),
                ("U", C.c_void_p * 2), ("ld", C.c_int * 2)]


class fc_params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("eps", C.c_double),
                ("tol_stop", C.c_double), ("eps_D", C.c_double), ("kmax", C.c_int),
                ("precond_rank", C.c_int), ("op_rank", C.c_int), ("rank_cap", C.c_int),
                ("boundary", C.c_int), ("precond_case", C.c_int)]


class fc_trunc_info(C.Structure):
    _fields_ = [("tucker_rank", C.c_int * 3), ("out_rank", C.c_int), ("required_rank", C.c_int),
                ("in_rank", C.c_int), ("basis_dim", C.c_int * 3), ("t2c_mode", C.c_int),
                ("energy", C.c_double), ("min_cut_margin", C.c_double)]


class fc_pcg_report(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("status", C.c_int),
                ("rel_res", C.c_double * FC_MAX_ITERS),
                ("rank_X", C.c_int * FC_MAX_ITERS), ("rank_R", C.c_int * FC_MAX_ITERS),
                ("rank_Z", C.c_int * FC_MAX_ITERS), ("rank_P", C.c_int * FC_MAX_ITERS),
                ("rank_S", C.c_int * FC_MAX_ITERS), ("tucker_S", C.c_int * FC_MAX_ITERS),
                ("t_iter_ms", C.c_double * FC_MAX_ITERS), ("t_total_ms", C.c_double),
                ("t_loop_ms", C.c_double), ("normB", C.c_double), ("cap_hits", C.c_int)]

    def as_dict(self):
        k = self.iters
        return {"iters": k, "converged": bool(self.converged), "status": STATUS.get(self.status, self.status),
                "rel_res": list(self.rel_res[:k]), "rank_X": list(self.rank_X[:k]),
                "rank_R": list(self.rank_R[:k]), "rank_Z": list(self.rank_Z[:k]),
                "rank_P": list(self.rank_P[:k]), "rank_S": list(self.rank_S[:k]),
                "tucker_S": list(self.tucker_S[:k]), "t_iter_ms": list(self.t_iter_ms[:k]),
                "t_total_ms": self.t_total_ms, "t_loop_ms": self.t_loop_ms, "normB": self.normB,
                "cap_hits": self.cap_hits}


class FCError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)} ({code}): {msg}")
        self.code = code


ENTRY_POINTS = ["fc_create", "fc_destroy", "fc_last_error", "fc_set_stream", "sl_setup", "sl_get_eigen",
                "sl_set_eigen", "op_get_spectral_cp", "op_set_spectral_cp", "op_spectral_rank",
                "fracop_apply", "precond_apply", "cp_dot", "cp_axpy", "cp_truncate", "pcg_solve",
                "fc_dgemm", "fc_dgemm_splitk", "fc_dgemm_streamk", "fc_last_kernel_stats", "fc_kernel_launches", "fracop_apply_truncate", "fc_orthonormalize",
                "fc_profile_gemm", "fc_profile_kernel", "fc_syev", "op_get_precond_basis", "op_set_precond_basis", "state_recover", "op_build_spectral_sinc",
                "sl_setup_2d", "op_get_spectral_2d", "op_set_spectral_2d", "fracop_apply_2d", "cp_dot_2d",
                "cp_truncate_2d", "pcg_solve_2d", "cp_truncate_als"]


def load_library(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built: run `python -m paper_2006_09314_b200.build` "
                                "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, I, D = C.c_void_p, C.c_int, C.c_double
    cpp = C.POINTER(fc_cp)
    sig = {
        "fc_create": ([C.POINTER(P), P], I), "fc_destroy": ([P], I), "fc_last_error": ([P], C.c_char_p),
        "fc_set_stream": ([P, P], I),
        "sl_setup": ([P, I, P, C.POINTER(fc_params)], I),
        "sl_get_eigen": ([P, I, P, P], I),
        "sl_set_eigen": ([P, I, I, P, P, C.POINTER(fc_params)], I),
        "op_get_spectral_cp": ([P, I, cpp], I), "op_set_spectral_cp": ([P, I, cpp], I),
        "op_spectral_rank": ([P, I, C.POINTER(I), P], I),
        "fracop_apply": ([P, I, cpp, cpp], I), "precond_apply": ([P, cpp, cpp], I),
        "cp_dot": ([P, cpp, cpp, C.POINTER(D)], I), "cp_axpy": ([P, cpp, D, cpp, cpp], I),
        "cp_truncate": ([P, cpp, D, cpp, C.POINTER(fc_trunc_info)], I),
        "fracop_apply_truncate": ([P, I, cpp, D, cpp, C.POINTER(fc_trunc_info)], I),
        "pcg_solve": ([P, cpp, C.POINTER(fc_params), cpp, C.POINTER(fc_pcg_report)], I),
        "fc_dgemm": ([P, I, I, I, I, I, D, P, I, P, I, D, P, I], I),
        "fc_dgemm_splitk": ([P, I, I, I, I, I, D, P, I, P, I, D, P, I, I], I),
        "fc_dgemm_streamk": ([P, I, I, I, I, I, D, P, I, P, I, D, P, I], I),
        "fc_last_kernel_stats": ([P, C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(I)], I),
        "fc_kernel_launches": ([C.POINTER(C.c_longlong)], I),
        "fc_orthonormalize": ([P, I, I, P, P, D, C.POINTER(I)], I),
        "fc_profile_gemm": ([P, I, C.POINTER(D), C.POINTER(D), C.POINTER(C.c_longlong)], I),
        "fc_profile_kernel": ([P, I, I, C.POINTER(D), C.POINTER(D), C.POINTER(C.c_longlong)], I),
        "fc_syev": ([P, I, C.POINTER(I), C.POINTER(P), C.POINTER(I), C.POINTER(P), C.POINTER(P), C.POINTER(I),
                     C.POINTER(I)], I),
        "op_get_precond_basis": ([P, I, P, P], I), "op_set_precond_basis": ([P, I, P, P], I),
        "state_recover": ([P, cpp, D, cpp, C.POINTER(fc_trunc_info)], I),
        "op_build_spectral_sinc": ([P, I, D], I),
        "cp_truncate_als": ([P, cpp, D, I, cpp, C.POINTER(fc_trunc_info)], I),
        "sl_setup_2d": ([P, I, P, C.POINTER(fc_params)], I),
        "op_get_spectral_2d": ([P, I, C.POINTER(fc_lr2)], I), "op_set_spectral_2d": ([P, I, C.POINTER(fc_lr2)], I),
        "fracop_apply_2d": ([P, I, C.POINTER(fc_lr2), C.POINTER(fc_lr2)], I),
        "cp_dot_2d": ([P, C.POINTER(fc_lr2), C.POINTER(fc_lr2), C.POINTER(D)], I),
        "cp_truncate_2d": ([P, C.POINTER(fc_lr2), D, C.POINTER(fc_lr2), C.POINTER(I)], I),
        "pcg_solve_2d": ([P, C.POINTER(fc_lr2), C.POINTER(fc_params), C.POINTER(fc_lr2), C.POINTER(fc_pcg_report)], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


def make_params(alpha, beta, eps, tol_stop=0.0, eps_D=0.0, kmax=0, precond_rank=0, op_rank=0,
                rank_cap=0, boundary=0, precond_case=FC_PRECOND_B) -> fc_params:
    return fc_params(alpha, beta, eps, tol_stop, eps_D, kmax, precond_rank, op_rank, rank_cap, boundary,
                     precond_case)


class DeviceCP:
    """A CP tensor in device memory: w (cap,), U[l] stored (cap, n) row-major = n x cap
    column-major with ld = n (the ABI layout)."""

    def __init__(self, n: int, cap: int, rank: int = 0, device="cuda"):
        import torch
        self.n, self.cap, self.rank = n, max(cap, 1), rank
        self.w = torch.zeros(self.cap, dtype=torch.float64, device=device)
        self.U = [torch.zeros(self.cap, n, dtype=torch.float64, device=device) for _ in range(3)]

    @classmethod
    def from_numpy(cls, w, U, cap=None, device="cuda"):
        import torch
        R = int(np.asarray(w).size)
        n = U[0].shape[0]
        x = cls(n, cap if cap is not None else R, R, device)
        x.w[:R] = torch.as_tensor(np.asarray(w, dtype=np.float64), device=device)
        for l in range(3):
            x.U[l][:R] = torch.as_tensor(np.ascontiguousarray(np.asarray(U[l], dtype=np.float64).T), device=device)
        return x

    def to_numpy(self):
        R = self.rank
        return (self.w[:R].cpu().numpy().copy(), [self.U[l][:R].cpu().numpy().T.copy() for l in range(3)])

    def struct(self) -> fc_cp:
        s = fc_cp()
        for l in range(3):
            s.n[l] = self.n
            s.U[l] = self.U[l].data_ptr()
            s.ld[l] = self.n
        s.rank, s.cap, s.w = self.rank, self.cap, self.w.data_ptr()
        return s


class DeviceLR2:
    """A 2D low-rank matrix in device memory (fc_lr2): w (cap,), U[l] stored (cap, n) row-major =
    n x cap column-major with ld = n."""

    def __init__(self, n: int, cap: int, rank: int = 0, device="cuda"):
        import torch
        self.n, self.cap, self.rank = n, max(cap, 1), rank
        self.w = torch.zeros(self.cap, dtype=torch.float64, device=device)
        self.U = [torch.zeros(self.cap, n, dtype=torch.float64, device=device) for _ in range(2)]

    @classmethod
    def from_numpy(cls, w, U, cap=None, device="cuda"):
        import torch
        R = int(np.asarray(w).size)
        n = U[0].shape[0]
        x = cls(n, cap if cap is not None else R, R, device)
        x.w[:R] = torch.as_tensor(np.asarray(w, dtype=np.float64), device=device)
        for l in range(2):
            x.U[l][:R] = torch.as_tensor(np.ascontiguousarray(np.asarray(U[l], dtype=np.float64).T), device=device)
        return x

    def to_numpy(self):
        R = self.rank
        return (self.w[:R].cpu().numpy().copy(), [self.U[l][:R].cpu().numpy().T.copy() for l in range(2)])

    def struct(self) -> fc_lr2:
        s = fc_lr2()
        for l in range(2):
            s.n[l] = self.n
            s.U[l] = self.U[l].data_ptr()
            s.ld[l] = self.n
        s.rank, s.cap, s.w = self.rank, self.cap, self.w.data_ptr()
        return s


class Library:
    def __init__(self, path: str = LIB_PATH):
        self.lib = load_library(path)

    def context(self, stream=None) -> "Context":
        return Context(self, stream)


def kernel_launches(L: "Library") -> int:
    v = C.c_longlong()
    L.lib.fc_kernel_launches(C.byref(v))
    return v.value


class Context:
    def __init__(self, L: Library, stream=None):
        import torch
        self.L, self.lib = L, L.lib
        self.h = C.c_void_p()
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        self._check(self.lib.fc_create(C.byref(self.h), C.c_void_p(s)))
        self.n = 0

    def __del__(self):
        try:
            if self.h:
                self.lib.fc_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def _check(self, rc, ok=(0,)):
        if rc not in ok:
            msg = self.lib.fc_last_error(self.h).decode() if getattr(self, "h", None) else ""
            raise FCError(rc, msg)
        return rc

    # ---- setup ----
    def sl_setup(self, n, a_mid, params: fc_params):
        a = np.ascontiguousarray(np.asarray(a_mid, dtype=np.float64).reshape(3, n + 1))
        self._check(self.lib.sl_setup(self.h, n, a.ctypes.data, C.byref(params)))
        self.n = n

    def sl_get_eigen(self, mode):
        import torch
        lam = torch.empty(self.n, dtype=torch.float64, device="cuda")
        Vt = torch.empty(self.n, self.n, dtype=torch.float64, device="cuda")   # (col, row) = V^T row-major
        self._check(self.lib.sl_get_eigen(self.h, mode, lam.data_ptr(), Vt.data_ptr()))
        return lam, Vt.T

    def op_get_precond_basis(self, mode):
        import torch
        lam = torch.empty(self.n, dtype=torch.float64, device="cuda")
        Vt = torch.empty(self.n, self.n, dtype=torch.float64, device="cuda")
        self._check(self.lib.op_get_precond_basis(self.h, mode, lam.data_ptr(), Vt.data_ptr()))
        return lam, Vt.T

    def op_set_precond_basis(self, mode, lam, V):
        import torch
        lam_t = torch.as_tensor(np.asarray(lam, dtype=np.float64), device="cuda").contiguous()
        Vt = torch.as_tensor(np.ascontiguousarray(np.asarray(V, dtype=np.float64).T), device="cuda")
        self._check(self.lib.op_set_precond_basis(self.h, mode, lam_t.data_ptr(), Vt.data_ptr()))

    def sl_set_eigen(self, n, mode, lam, V, params: fc_params | None = None):
        import torch
        lam_t = torch.as_tensor(np.asarray(lam, dtype=np.float64), device="cuda").contiguous()
        Vt = torch.as_tensor(np.ascontiguousarray(np.asarray(V, dtype=np.float64).T), device="cuda")
        self._check(self.lib.sl_set_eigen(self.h, n, mode, lam_t.data_ptr(), Vt.data_ptr(),
                                          C.byref(params) if params is not None else None))
        self.n = n

    def op_set_spectral_cp(self, which, x: DeviceCP):
        s = x.struct()
        self._check(self.lib.op_set_spectral_cp(self.h, which, C.byref(s)))

    def op_spectral_rank(self, which):
        r = C.c_int()
        t = (C.c_int * 3)()
        self._check(self.lib.op_spectral_rank(self.h, which, C.byref(r), t))
        return r.value, list(t)

    def op_get_spectral_cp(self, which) -> DeviceCP:
        r, _ = self.op_spectral_rank(which)
        y = DeviceCP(self.n, r)
        s = y.struct()
        self._check(self.lib.op_get_spectral_cp(self.h, which, C.byref(s)))
        y.rank = s.rank
        return y

    # ---- operator ----
    def fracop_apply(self, which, x: DeviceCP, y: DeviceCP | None = None) -> DeviceCP:
        if y is None:
            r, _ = self.op_spectral_rank(which)
            y = DeviceCP(self.n, r * x.rank)
        xs, ys = x.struct(), y.struct()
        self._check(self.lib.fracop_apply(self.h, which, C.byref(xs), C.byref(ys)))
        y.rank = ys.rank
        return y

    def precond_apply(self, x, y=None):
        return self.fracop_apply(FC_G, x, y)

    def cp_dot(self, x: DeviceCP, y: DeviceCP) -> float:
        out = C.c_double()
        xs, ys = x.struct(), y.struct()
        self._check(self.lib.cp_dot(self.h, C.byref(xs), C.byref(ys), C.byref(out)))
        return out.value

    def cp_axpy(self, x, a, y, z=None):
        if z is None:
            z = DeviceCP(self.n, x.rank + y.rank)
        xs, ys, zs = x.struct(), y.struct(), z.struct()
        self._check(self.lib.cp_axpy(self.h, C.byref(xs), C.c_double(a), C.byref(ys), C.byref(zs)))
        z.rank = zs.rank
        return z

    def cp_truncate(self, x: DeviceCP, eps: float, cap: int | None = None):
        cap = cap if cap is not None else max(4 * x.rank, 64)
        while True:
            y = DeviceCP(self.n, cap)
            info = fc_trunc_info()
            xs, ys = x.struct(), y.struct()
            rc = self.lib.cp_truncate(self.h, C.byref(xs), C.c_double(eps), C.byref(ys), C.byref(info))
            if rc == -3 and info.required_rank > cap:
                cap = info.required_rank
                continue
            self._check(rc)
            y.rank = ys.rank
            return y, info

    def cp_truncate_als(self, x: DeviceCP, eps: float, sweeps: int = 2, cap: int | None = None):
        cap = cap if cap is not None else max(4 * x.rank, 64)
        while True:
            y = DeviceCP(self.n, cap)
            info = fc_trunc_info()
            xs, ys = x.struct(), y.struct()
            rc = self.lib.cp_truncate_als(self.h, C.byref(xs), C.c_double(eps), sweeps, C.byref(ys), C.byref(info))
            if rc == -3 and info.required_rank > cap:
                cap = info.required_rank
                continue
            self._check(rc)
            y.rank = ys.rank
            return y, info

    def fracop_apply_truncate(self, which, x: DeviceCP, eps: float, cap: int | None = None):
        cap = cap if cap is not None else max(4 * x.rank, 64)
        while True:
            y = DeviceCP(self.n, cap)
            info = fc_trunc_info()
            xs, ys = x.struct(), y.struct()
            rc = self.lib.fracop_apply_truncate(self.h, which, C.byref(xs), C.c_double(eps), C.byref(ys),
                                                C.byref(info))
            if rc == -3 and info.required_rank > cap:
                cap = info.required_rank
                continue
            self._check(rc)
            y.rank = ys.rank
            return y, info

    def op_build_spectral_sinc(self, which, eps):
        self._check(self.lib.op_build_spectral_sinc(self.h, which, C.c_double(eps)))

    def state_recover(self, u: DeviceCP, eps: float, cap: int | None = None):
        """y = A^-alpha u truncated at eps (state_recover)."""
        cap = cap if cap is not None else max(4 * u.rank, 64)
        while True:
            y = DeviceCP(self.n, cap)
            info = fc_trunc_info()
            us, ys = u.struct(), y.struct()
            rc = self.lib.state_recover(self.h, C.byref(us), C.c_double(eps), C.byref(ys), C.byref(info))
            if rc == -3 and info.required_rank > cap:
                cap = info.required_rank
                continue
            self._check(rc)
            y.rank = ys.rank
            return y, info

    def pcg_solve(self, b: DeviceCP, params: fc_params, cap: int = 4096, u: DeviceCP | None = None):
        while True:
            if u is None or u.cap < cap:
                u = DeviceCP(self.n, cap)
            rep = fc_pcg_report()
            bs, us = b.struct(), u.struct()
            rc = self.lib.pcg_solve(self.h, C.byref(bs), C.byref(params), C.byref(us), C.byref(rep))
            if rc == -3 and us.rank > u.cap:        # the solution's rank exceeds u.cap: re-run
                cap = us.rank
                continue
            self._check(rc, ok=(0, 1, 2))
            u.rank = us.rank
            return u, rep.as_dict(), rc

    # ---- 2D variant ----
    def sl_setup_2d(self, n, a_mid, params: fc_params):
        a = np.ascontiguousarray(np.asarray(a_mid, dtype=np.float64).reshape(2, n + 1))
        self._check(self.lib.sl_setup_2d(self.h, n, a.ctypes.data, C.byref(params)))
        self.n = n

    def op_get_spectral_2d(self, which, cap: int = 128) -> DeviceLR2:
        while True:
            y = DeviceLR2(self.n, cap)
            s = y.struct()
            rc = self.lib.op_get_spectral_2d(self.h, which, C.byref(s))
            if rc == -3 and s.rank > cap:
                cap = s.rank
                continue
            self._check(rc)
            y.rank = s.rank
            return y

    def op_set_spectral_2d(self, which, x: DeviceLR2):
        s = x.struct()
        self._check(self.lib.op_set_spectral_2d(self.h, which, C.byref(s)))

    def fracop_apply_2d(self, which, x: DeviceLR2, cap: int | None = None) -> DeviceLR2:
        cap = cap if cap is not None else 64 * max(x.rank, 1)
        while True:
            y = DeviceLR2(self.n, cap)
            xs, ys = x.struct(), y.struct()
            rc = self.lib.fracop_apply_2d(self.h, which, C.byref(xs), C.byref(ys))
            if rc == -3 and ys.rank > cap:
                cap = ys.rank
                continue
            self._check(rc)
            y.rank = ys.rank
            return y

    def cp_dot_2d(self, x: DeviceLR2, y: DeviceLR2) -> float:
        out = C.c_double()
        xs, ys = x.struct(), y.struct()
        self._check(self.lib.cp_dot_2d(self.h, C.byref(xs), C.byref(ys), C.byref(out)))
        return out.value

    def cp_truncate_2d(self, x: DeviceLR2, eps: float, cap: int | None = None):
        cap = cap if cap is not None else max(x.rank, 16)
        while True:
            y = DeviceLR2(self.n, cap)
            r = C.c_int()
            xs, ys = x.struct(), y.struct()
            rc = self.lib.cp_truncate_2d(self.h, C.byref(xs), C.c_double(eps), C.byref(ys), C.byref(r))
            if rc == -3 and r.value > cap:
                cap = r.value
                continue
            self._check(rc)
            y.rank = ys.rank
            return y

    def pcg_solve_2d(self, b: DeviceLR2, params: fc_params, cap: int = 1024, u: DeviceLR2 | None = None):
        while True:
            if u is None or u.cap < cap:
                u = DeviceLR2(self.n, cap)
            rep = fc_pcg_report()
            bs, us = b.struct(), u.struct()
            rc = self.lib.pcg_solve_2d(self.h, C.byref(bs), C.byref(params), C.byref(us), C.byref(rep))
            if rc == -3 and us.rank > u.cap:
                cap = us.rank
                continue
            self._check(rc, ok=(0, 1, 2))
            u.rank = us.rank
            return u, rep.as_dict(), rc

    # ---- raw ----
    def profile_gemm(self, enable: bool):
        ms, fl, nl = C.c_double(), C.c_double(), C.c_longlong()
        self._check(self.lib.fc_profile_gemm(self.h, 1 if enable else 0, C.byref(ms), C.byref(fl), C.byref(nl)))
        return {"ms": ms.value, "flops": fl.value, "launches": nl.value}

    def profile_kernel(self, kernel: int, enable: bool):
        ms, b, nl = C.c_double(), C.c_double(), C.c_longlong()
        self._check(self.lib.fc_profile_kernel(self.h, kernel, 1 if enable else 0, C.byref(ms), C.byref(b),
                                               C.byref(nl)))
        return {"ms": ms.value, "bytes": b.value, "launches": nl.value}

    def orthonormalize(self, A, tau=1e-13):
        """A: torch (p, n) row-major == n x p column-major (overwritten).  Returns Q (k, n)."""
        import torch
        p, n = A.shape
        Q = torch.zeros(min(n, p), n, dtype=torch.float64, device=A.device)
        k = C.c_int()
        self._check(self.lib.fc_orthonormalize(self.h, n, p, A.data_ptr(), Q.data_ptr(), C.c_double(tau),
                                               C.byref(k)))
        return Q[:k.value]

    def syev(self, mats, rs):
        """Batched symmetric eigensolver (fc_syev).  mats: list of symmetric torch (N, N) float64
        CUDA tensors (overwritten); rs: wanted leading eigenvectors per matrix.  Returns
        [(lam descending (N,), Y (r, N) row-major == N x r column-major)]."""
        import torch
        nb = len(mats)
        Ns = [m.shape[0] for m in mats]
        lams = [torch.zeros(N, dtype=torch.float64, device=m.device) for N, m in zip(Ns, mats)]
        Ys = [torch.zeros(max(r, 1), N, dtype=torch.float64, device=m.device) for N, r, m in zip(Ns, rs, mats)]
        IA, PA = C.c_int * nb, C.c_void_p * nb
        self._check(self.lib.fc_syev(self.h, nb, IA(*Ns), PA(*[m.data_ptr() for m in mats]), IA(*Ns),
                                     PA(*[x.data_ptr() for x in lams]), PA(*[y.data_ptr() for y in Ys]),
                                     IA(*Ns), IA(*rs)))
        return [(lam, Y[:r]) for lam, Y, r in zip(lams, Ys, rs)]

    def dgemm(self, transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, Cm, ldc, splitk=None, streamk=False):
        if streamk:
            self._check(self.lib.fc_dgemm_streamk(self.h, transA, transB, M, N, K, alpha, A.data_ptr(), lda,
                                                  B.data_ptr(), ldb, beta, Cm.data_ptr(), ldc))
        elif splitk is None:
            self._check(self.lib.fc_dgemm(self.h, transA, transB, M, N, K, alpha, A.data_ptr(), lda,
                                          B.data_ptr(), ldb, beta, Cm.data_ptr(), ldc))
        else:
            self._check(self.lib.fc_dgemm_splitk(self.h, transA, transB, M, N, K, alpha, A.data_ptr(), lda,
                                                 B.data_ptr(), ldb, beta, Cm.data_ptr(), ldc, splitk))

    def last_kernel_stats(self):
        ms, fl, by, nl = C.c_double(), C.c_double(), C.c_double(), C.c_int()
        self._check(self.lib.fc_last_kernel_stats(self.h, C.byref(ms), C.byref(fl), C.byref(by), C.byref(nl)))
        return {"ms": ms.value, "flops": fl.value, "bytes": by.value, "launches": nl.value}
