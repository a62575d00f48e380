"""Thin Python binding of libredhess.so (include/redhess.h).

Argument marshalling only: every step of the reduced-Hessian path runs in the
library's sm_100a kernels.  Device arrays are torch CUDA tensors (fp64,
contiguous); streams are torch.cuda streams (default: the current stream).
There is no CPU fallback: importing this package without the built library
raises, and compute calls on a machine without a GPU raise RHError.

Method names follow the C ABI (rh_<name> -> RedHess.<name>).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libredhess.so")

(RH_OK, RH_E_ARG, RH_E_GRID, RH_E_ORDER, RH_E_SINGULAR, RH_E_CUDA, RH_E_NOMEM, RH_E_NODEV, RH_E_NOCONV,
 RH_E_NOTPD) = range(10)
STATUS_NAMES = {0: "RH_OK", 1: "RH_E_ARG", 2: "RH_E_GRID", 3: "RH_E_ORDER", 4: "RH_E_SINGULAR",
                5: "RH_E_CUDA", 6: "RH_E_NOMEM", 7: "RH_E_NODEV", 8: "RH_E_NOCONV", 9: "RH_E_NOTPD"}
KIND_THETA, KIND_V, KIND_PG = 0, 1, 2
JAC_ANALYTIC, JAC_COLORED = 0, 1

# every symbol declared in include/redhess.h (checked by tests/test_abi.py)
EXPORTS = ["rh_create", "rh_destroy", "rh_last_error", "rh_load_grid", "rh_get_info", "rh_orderings",
           "rh_symbolic", "rh_segments", "rh_set_state", "rh_residual", "rh_reduced_gradient", "rh_set_multipliers",
           "rh_newton",
           "rh_hvp", "rh_hvp_stages", "rh_hessian_columns", "rh_full_hessian", "rh_reduced_hessian",
           "rh_reduced_hessian_host", "rh_set_loads", "rh_dense_spd_solve", "rh_tracking_step",
           "rh_set_jacobian_mode", "rh_coloring", "rh_compressed_jacobian",
           "rh_launch_count", "rh_set_timing", "rh_stage_times", "rh_pivot_ratio"]


class RHError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


class rh_grid(ctypes.Structure):
    _fields_ = [("n_bus", ctypes.c_int32), ("n_line", ctypes.c_int32), ("n_gen", ctypes.c_int32),
                ("bus_type", ctypes.c_void_p), ("G_ii", ctypes.c_void_p), ("B_ii", ctypes.c_void_p),
                ("Pd", ctypes.c_void_p), ("Qd", ctypes.c_void_p), ("line_f", ctypes.c_void_p),
                ("line_t", ctypes.c_void_p), ("G_ft", ctypes.c_void_p), ("B_ft", ctypes.c_void_p),
                ("G_tf", ctypes.c_void_p), ("B_tf", ctypes.c_void_p), ("gen_bus", ctypes.c_void_p),
                ("c2", ctypes.c_void_p), ("c1", ctypes.c_void_p), ("c0", ctypes.c_void_p),
                ("theta_ref", ctypes.c_double)]


class rh_info(ctypes.Structure):
    _fields_ = [("n_bus", ctypes.c_int32), ("n_line", ctypes.c_int32), ("n_x", ctypes.c_int32),
                ("n_p", ctypes.c_int32), ("nnz_J", ctypes.c_int32), ("nnz_Gp", ctypes.c_int32),
                ("nnz_LU", ctypes.c_int32), ("levels_fwd", ctypes.c_int32), ("levels_bwd", ctypes.c_int32),
                ("max_level_rows", ctypes.c_int32), ("n_blocks", ctypes.c_int32), ("sep_rows", ctypes.c_int32),
                ("seg_levels", ctypes.c_int32), ("workspace_bytes", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2201_00241_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "rh_create": ([ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "rh_destroy": ([vp], ctypes.c_int),
        "rh_last_error": ([vp], ctypes.c_char_p),
        "rh_load_grid": ([vp, ctypes.POINTER(rh_grid), ctypes.POINTER(i32), ctypes.POINTER(i32)], ctypes.c_int),
        "rh_get_info": ([vp, ctypes.POINTER(rh_info)], ctypes.c_int),
        "rh_orderings": ([vp, vp, vp, vp, vp], ctypes.c_int),
        "rh_symbolic": ([vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "rh_segments": ([vp, vp], ctypes.c_int),
        "rh_set_state": ([vp, vp, vp, vp], ctypes.c_int),
        "rh_residual": ([vp, vp, vp, vp], ctypes.c_int),
        "rh_reduced_gradient": ([vp, vp, vp, vp], ctypes.c_int),
        "rh_set_multipliers": ([vp, vp, vp], ctypes.c_int),
        "rh_newton": ([vp, vp, vp, dbl, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(dbl), vp], ctypes.c_int),
        "rh_hvp": ([vp, vp, i64, vp, i64, i32, vp], ctypes.c_int),
        "rh_hvp_stages": ([vp, vp, i64, vp, i64, i32, vp, vp, vp, i64, vp], ctypes.c_int),
        "rh_hessian_columns": ([vp, i32, i32, i32, vp, i64, i32, vp], ctypes.c_int),
        "rh_full_hessian": ([vp, i32, vp, vp], ctypes.c_int),
        "rh_reduced_hessian": ([vp, vp, vp, i32, i32, i32, vp, vp, i64, i32, vp], ctypes.c_int),
        "rh_reduced_hessian_host": ([vp, vp, vp, i32, vp, vp], ctypes.c_int),
        "rh_set_loads": ([vp, vp, vp, vp], ctypes.c_int),
        "rh_dense_spd_solve": ([vp, i32, vp, i64, vp, vp, vp, dbl, ctypes.POINTER(dbl), ctypes.POINTER(i32), vp],
                               ctypes.c_int),
        "rh_tracking_step": ([vp, vp, vp, vp, vp, i32, i32, i32, dbl, vp, vp, i64, vp, vp, vp], ctypes.c_int),
        "rh_set_jacobian_mode": ([vp, i32], ctypes.c_int),
        "rh_coloring": ([vp, vp, ctypes.POINTER(i32)], ctypes.c_int),
        "rh_compressed_jacobian": ([vp, vp, vp], ctypes.c_int),
        "rh_launch_count": ([vp], i64),
        "rh_set_timing": ([vp, ctypes.c_int], ctypes.c_int),
        "rh_stage_times": ([vp, vp], ctypes.c_int),
        "rh_pivot_ratio": ([vp, vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    del dbl
    return lib


_LIB = None


def lib():
    """The loaded libredhess.so (raises ImportError if it is missing: no CPU fallback)."""
    global _LIB
    if _LIB is None:
        _LIB = _load()
    return _LIB


def _ptr(a):
    """Raw pointer of a numpy array or a torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check_dev(t, n=None, name="array", device=None):
    """A contiguous float64 CUDA tensor with exactly n elements (n=None: any size)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
    if device is not None and device >= 0 and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the context is on cuda:{device}")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} has {t.numel()} elements, need {n}")


def _check_dev_mat(t, rows, cols, name="array", device=None):
    """A row-major float64 CUDA matrix of shape [rows][cols] with unit column
    stride and row stride >= cols (the library's [row][ld] layout)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a float64 CUDA tensor")
    if device is not None and device >= 0 and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the context is on cuda:{device}")
    if t.dim() != 2 or tuple(t.shape) != (rows, cols):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, need ({rows}, {cols})")
    if cols > 0 and rows > 0 and (t.stride(1) != 1 or t.stride(0) < cols):
        raise ValueError(f"{name} must be row-major with unit column stride (strides {t.stride()})")


def _check_host(a, shape, name="array", writable=False):
    """A C-contiguous float64 HOST array (numpy, or a CPU torch tensor) of exactly `shape`."""
    if isinstance(a, np.ndarray):
        ok = a.dtype == np.float64 and a.flags.c_contiguous and (a.flags.writeable or not writable)
        shp = a.shape
    else:
        import torch
        if not isinstance(a, torch.Tensor) or a.is_cuda:
            raise TypeError(f"{name} must be a host (numpy or CPU torch) float64 array")
        ok = a.dtype == torch.float64 and a.is_contiguous()
        shp = tuple(a.shape)
    if not ok:
        raise TypeError(f"{name} must be a C-contiguous{' writable' if writable else ''} float64 host array")
    if tuple(shp) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(shp)}, need {tuple(shape)}")


class RedHess:
    """One rh_ctx.  device=-1 gives a host-only context (analysis only)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        rc = lib().rh_create(int(device), ctypes.byref(h))
        if rc != RH_OK:
            raise RHError(rc, f"rh_create(device={device}) failed")
        self._h = h
        self.device = device
        self.n_x = self.n_p = None
        self._keep = None

    def close(self):
        if getattr(self, "_h", None):
            lib().rh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _rc(self, rc):
        if rc != RH_OK:
            raise RHError(rc, lib().rh_last_error(self._h).decode())

    # ------------------------------------------------------------------ grid
    def load_grid(self, grid):
        """grid: any object with the rh_grid fields as numpy arrays (gridgen.Grid)."""
        keep = dict(
            bus_type=np.ascontiguousarray(grid.bus_type, np.int32),
            G_ii=np.ascontiguousarray(grid.G_ii, np.float64), B_ii=np.ascontiguousarray(grid.B_ii, np.float64),
            Pd=np.ascontiguousarray(grid.Pd, np.float64), Qd=np.ascontiguousarray(grid.Qd, np.float64),
            line_f=np.ascontiguousarray(grid.line_f, np.int32), line_t=np.ascontiguousarray(grid.line_t, np.int32),
            G_ft=np.ascontiguousarray(grid.G_ft, np.float64), B_ft=np.ascontiguousarray(grid.B_ft, np.float64),
            G_tf=np.ascontiguousarray(grid.G_tf, np.float64), B_tf=np.ascontiguousarray(grid.B_tf, np.float64),
            gen_bus=np.ascontiguousarray(grid.gen_bus, np.int32), c2=np.ascontiguousarray(grid.c2, np.float64),
            c1=np.ascontiguousarray(grid.c1, np.float64), c0=np.ascontiguousarray(grid.c0, np.float64))
        g = rh_grid(n_bus=keep["bus_type"].shape[0], n_line=keep["line_f"].shape[0],
                    n_gen=keep["gen_bus"].shape[0], theta_ref=float(grid.theta_ref),
                    **{k: v.ctypes.data for k, v in keep.items()})
        nx, npp = ctypes.c_int32(), ctypes.c_int32()
        self._rc(lib().rh_load_grid(self._h, ctypes.byref(g), ctypes.byref(nx), ctypes.byref(npp)))
        self.n_x, self.n_p = nx.value, npp.value
        self.n_bus = int(g.n_bus)
        return self.n_x, self.n_p

    def get_info(self):
        info = rh_info()
        self._rc(lib().rh_get_info(self._h, ctypes.byref(info)))
        return {k: getattr(info, k) for k, _ in rh_info._fields_}

    def orderings(self):
        xb, xk = np.zeros(self.n_x, np.int32), np.zeros(self.n_x, np.int32)
        pb, pk = np.zeros(self.n_p, np.int32), np.zeros(self.n_p, np.int32)
        self._rc(lib().rh_orderings(self._h, _ptr(xb), _ptr(xk), _ptr(pb), _ptr(pk)))
        return xb, xk, pb, pk

    def symbolic(self):
        info = self.get_info()
        perm = np.zeros(self.n_x, np.int32)
        rp = np.zeros(self.n_x + 1, np.int32)
        ci = np.zeros(info["nnz_LU"], np.int32)
        lf = np.zeros(self.n_x, np.int32)
        lb = np.zeros(self.n_x, np.int32)
        self._rc(lib().rh_symbolic(self._h, _ptr(perm), _ptr(rp), _ptr(ci), _ptr(lf), _ptr(lb)))
        seg = np.zeros(self.n_x, np.int32)
        self._rc(lib().rh_segments(self._h, _ptr(seg)))
        return dict(perm=perm, rowptr=rp, colidx=ci, level_fwd=lf, level_bwd=lb, segment=seg)

    def state_vectors(self, grid):
        """x, p (numpy) from the grid's bus-level theta, v, Pg in this library's orderings."""
        xb, xk, pb, pk = self.orderings()
        th, v = np.asarray(grid.theta), np.asarray(grid.v)
        x = np.where(xk == KIND_THETA, th[xb], v[xb]).astype(np.float64)
        pg_of_bus = np.zeros(th.shape[0])
        pg_of_bus[np.asarray(grid.gen_bus)] = grid.Pg
        p = np.where(pk == KIND_PG, pg_of_bus[pb], v[pb]).astype(np.float64)
        return x, p

    # ------------------------------------------------------------------ compute (device)
    def set_state(self, x, p, stream=None):
        _check_dev(x, self.n_x, "x", self.device)
        _check_dev(p, self.n_p, "p", self.device)
        self._rc(lib().rh_set_state(self._h, _ptr(x), _ptr(p), _stream(stream)))

    def residual(self, g=None, f=None, stream=None):
        import torch
        g = torch.empty(self.n_x, dtype=torch.float64, device="cuda") if g is None else g
        f = torch.empty(1, dtype=torch.float64, device="cuda") if f is None else f
        _check_dev(g, self.n_x, "g", self.device)
        _check_dev(f, 1, "f", self.device)
        self._rc(lib().rh_residual(self._h, _ptr(g), _ptr(f), _stream(stream)))
        return g, f

    def reduced_gradient(self, grad=None, lam=None, stream=None):
        import torch
        grad = torch.empty(self.n_p, dtype=torch.float64, device="cuda") if grad is None else grad
        lam = torch.empty(self.n_x, dtype=torch.float64, device="cuda") if lam is None else lam
        _check_dev(grad, self.n_p, "grad", self.device)
        _check_dev(lam, self.n_x, "lambda", self.device)
        self._rc(lib().rh_reduced_gradient(self._h, _ptr(grad), _ptr(lam), _stream(stream)))
        return grad, lam

    def set_multipliers(self, lam, stream=None):
        _check_dev(lam, self.n_x, "lambda", self.device)
        self._rc(lib().rh_set_multipliers(self._h, _ptr(lam), _stream(stream)))

    def hvp(self, W, HW=None, stream=None):
        """W: [n_p][N] float64 CUDA tensor (batch index fastest) -> HW [n_p][N]."""
        import torch
        if not isinstance(W, torch.Tensor) or W.dim() != 2:
            raise TypeError("W must be a 2-D float64 CUDA tensor [n_p][N]")
        N = W.shape[1]
        _check_dev_mat(W, self.n_p, N, "W", self.device)
        HW = torch.empty((self.n_p, N), dtype=torch.float64, device=W.device) if HW is None else HW
        _check_dev_mat(HW, self.n_p, N, "HW", self.device)
        self._rc(lib().rh_hvp(self._h, _ptr(W), W.stride(0), _ptr(HW), HW.stride(0), N, _stream(stream)))
        return HW

    def hvp_stages(self, W, stream=None):
        import torch
        if not isinstance(W, torch.Tensor) or W.dim() != 2:
            raise TypeError("W must be a 2-D float64 CUDA tensor [n_p][N]")
        N = W.shape[1]
        _check_dev_mat(W, self.n_p, N, "W", self.device)
        HW = torch.empty((self.n_p, N), dtype=torch.float64, device=W.device)
        Z, Yx, Psi = (torch.empty((self.n_x, N), dtype=torch.float64, device=W.device) for _ in range(3))
        self._rc(lib().rh_hvp_stages(self._h, _ptr(W), W.stride(0), _ptr(HW), HW.stride(0), N, _ptr(Z), _ptr(Yx),
                                    _ptr(Psi), Z.stride(0), _stream(stream)))
        return HW, Z, Yx, Psi

    def _check_range(self, j0, j1):
        if not (0 <= j0 <= j1 <= self.n_p):
            raise ValueError(f"column range [{j0}, {j1}) is not inside [0, {self.n_p})")

    def _cols_out(self, H, j0, j1, transposed):
        import torch
        shape = (j1 - j0, self.n_p) if transposed else (self.n_p, j1 - j0)
        if H is None:
            return torch.empty(shape, dtype=torch.float64, device="cuda")
        if j1 == j0:     # nothing is written; any float64 CUDA matrix will do
            if not isinstance(H, torch.Tensor) or not H.is_cuda or H.dtype != torch.float64 or H.dim() != 2:
                raise TypeError("H must be a float64 CUDA matrix")
            return H
        _check_dev_mat(H, shape[0], shape[1], "H", self.device)
        return H

    def hessian_columns(self, j0, j1, N, H=None, transposed=False, stream=None):
        self._check_range(j0, j1)
        H = self._cols_out(H, j0, j1, transposed)
        self._rc(lib().rh_hessian_columns(self._h, j0, j1, N, _ptr(H), H.stride(0), int(bool(transposed)),
                                         _stream(stream)))
        return H

    def full_hessian(self, N, H=None, stream=None):
        import torch
        H = torch.empty((self.n_p, self.n_p), dtype=torch.float64, device="cuda") if H is None else H
        _check_dev(H, self.n_p * self.n_p, "H", self.device)
        if H.dim() != 2 or tuple(H.shape) != (self.n_p, self.n_p):
            raise ValueError(f"H has shape {tuple(H.shape)}, need ({self.n_p}, {self.n_p})")
        self._rc(lib().rh_full_hessian(self._h, N, _ptr(H), _stream(stream)))
        return H

    # ------------------------------------------------------------------ compute (host buffers)
    def newton(self, x, p, tol=1e-11, extra=2, maxit=40, stream=None):
        """rh_newton: Newton-Raphson projection x(p) in place on the DEVICE vector x; returns (steps, max|g|)."""
        _check_dev(x, self.n_x, "x", self.device)
        _check_dev(p, self.n_p, "p", self.device)
        it = ctypes.c_int32(0)
        res = ctypes.c_double(0.0)
        self._rc(lib().rh_newton(self._h, _ptr(x), _ptr(p), float(tol), int(extra), int(maxit), ctypes.byref(it),
                                 ctypes.byref(res), _stream(stream)))
        return it.value, res.value

    def reduced_hessian(self, x, p, N, j0=0, j1=None, grad=None, H=None, transposed=False, stream=None):
        """rh_reduced_hessian: state + reduced gradient + Hessian columns [j0, j1) in one call (DEVICE)."""
        import torch
        j1 = self.n_p if j1 is None else j1
        self._check_range(j0, j1)
        _check_dev(x, self.n_x, "x", self.device)
        _check_dev(p, self.n_p, "p", self.device)
        if grad is None:
            grad = torch.empty(self.n_p, dtype=torch.float64, device="cuda")
        _check_dev(grad, self.n_p, "grad", self.device)
        H = self._cols_out(H, j0, j1, transposed)
        self._rc(lib().rh_reduced_hessian(self._h, _ptr(x), _ptr(p), j0, j1, N, _ptr(grad), _ptr(H), H.stride(0),
                                          int(bool(transposed)), _stream(stream)))
        return grad, H

    def reduced_hessian_host(self, x, p, N, grad=None, H=None):
        """End to end with HOST buffers (numpy or pinned torch CPU tensors)."""
        if H is None:
            H = np.empty((self.n_p, self.n_p))
        if grad is None:
            grad = np.empty(self.n_p)
        _check_host(x, (self.n_x,), "x")
        _check_host(p, (self.n_p,), "p")
        _check_host(grad, (self.n_p,), "grad", writable=True)
        _check_host(H, (self.n_p, self.n_p), "H", writable=True)
        self._rc(lib().rh_reduced_hessian_host(self._h, _ptr(x), _ptr(p), N, _ptr(grad), _ptr(H)))
        return grad, H

    # ------------------------------------------------------------------ real-time tracking (PAPER.md 6.3)
    def set_loads(self, Pd=None, Qd=None, stream=None):
        """rh_set_loads: DEVICE loads [n_bus] (None = keep); invalidates the state."""
        if Pd is not None:
            _check_dev(Pd, self.n_bus, "Pd", self.device)
        if Qd is not None:
            _check_dev(Qd, self.n_bus, "Qd", self.device)
        self._rc(lib().rh_set_loads(self._h, _ptr(Pd) if Pd is not None else None,
                                    _ptr(Qd) if Qd is not None else None, _stream(stream)))

    def dense_spd_solve(self, H, g, d=None, p=None, alpha=1.0, stream=None):
        """rh_dense_spd_solve: d with ((H + H^T)/2 + tau I) d = -g (Eq. qp_rto), DEVICE tensors;
        p += alpha d when p is given.  Returns (d, tau, attempts)."""
        import torch
        n = g.shape[0]
        _check_dev(g, n, "g", self.device)
        if (not isinstance(H, torch.Tensor) or not H.is_cuda or H.dim() != 2 or H.shape[0] < n or H.shape[1] < n
                or (n > 0 and H.stride(1) != 1) or H.dtype != torch.float64):
            raise ValueError("H must be a row-major float64 [>= n][>= n] CUDA matrix")
        if d is None:
            d = torch.empty(n, dtype=torch.float64, device=g.device)
        _check_dev(d, n, "d", self.device)
        if p is not None:
            _check_dev(p, n, "p", self.device)
        tau = ctypes.c_double(0.0)
        att = ctypes.c_int32(0)
        self._rc(lib().rh_dense_spd_solve(self._h, n, _ptr(H), H.stride(0), _ptr(g), _ptr(d),
                                          _ptr(p) if p is not None else None, float(alpha), ctypes.byref(tau),
                                          ctypes.byref(att), _stream(stream)))
        return d, tau.value, att.value

    def tracking_step(self, x, p, N, Pd=None, Qd=None, j0=0, j1=None, alpha=1.0, grad=None, H=None, d=None,
                      stream=None):
        """rh_tracking_step: x <- x(p; w), g_t, columns [j0, j1) of H_t
        (transposed), d = -H_ff^-1 g_f, p[j0:j1] += alpha d.  DEVICE x, p (updated in place).
        Returns (grad, H, d, info) with info = dict(newton_steps, resid, F, tau, attempts, ms_step1, ms_step2)."""
        import torch
        j1 = self.n_p if j1 is None else j1
        _check_dev(x, self.n_x, "x", self.device)
        _check_dev(p, self.n_p, "p", self.device)
        for name, v in (("Pd", Pd), ("Qd", Qd)):
            if v is not None:
                _check_dev(v, self.n_bus, name, self.device)
        self._check_range(j0, j1)
        if grad is None:
            grad = torch.empty(self.n_p, dtype=torch.float64, device="cuda")
        _check_dev(grad, self.n_p, "grad", self.device)
        H = self._cols_out(H, j0, j1, True)
        if d is None:
            d = torch.empty(j1 - j0, dtype=torch.float64, device="cuda")
        _check_dev(d, j1 - j0, "d", self.device)
        info = np.zeros(7)
        self._rc(lib().rh_tracking_step(self._h, _ptr(x), _ptr(p), _ptr(Pd) if Pd is not None else None,
                                        _ptr(Qd) if Qd is not None else None, j0, j1, N, float(alpha), _ptr(grad),
                                        _ptr(H), H.stride(0), _ptr(d), _ptr(info), _stream(stream)))
        keys = ("newton_steps", "resid", "F", "tau", "attempts", "ms_step1", "ms_step2")
        return grad, H, d, dict(zip(keys, info.tolist()))

    # ------------------------------------------------------------------ colored Jacobians (PAPER.md 4)
    def set_jacobian_mode(self, mode):
        """rh_set_jacobian_mode: JAC_ANALYTIC or JAC_COLORED (coloring + forward mode)."""
        self._rc(lib().rh_set_jacobian_mode(self._h, int(mode)))

    def coloring(self):
        """rh_coloring: (colors [n_x + n_p] int32, ncolors)."""
        nc = ctypes.c_int32(0)
        colors = np.zeros(self.n_x + self.n_p, np.int32)
        self._rc(lib().rh_coloring(self._h, _ptr(colors), ctypes.byref(nc)))
        return colors, nc.value

    def compressed_jacobian(self, stream=None):
        """rh_compressed_jacobian: JS [n_x][ncolors] (DEVICE) at the current state."""
        import torch
        _, nc = self.coloring()
        JS = torch.empty((self.n_x, max(1, nc)), dtype=torch.float64, device="cuda")
        self._rc(lib().rh_compressed_jacobian(self._h, _ptr(JS), _stream(stream)))
        return JS

    # ------------------------------------------------------------------ accounting
    def launch_count(self):
        return int(lib().rh_launch_count(self._h))

    def set_timing(self, enable=True):
        self._rc(lib().rh_set_timing(self._h, int(bool(enable))))

    def pivot_ratio(self):
        """rh_pivot_ratio: smallest |u_kk| / max|J row k| of the last refactorization (R15)."""
        out = np.zeros(1, np.float64)
        self._rc(lib().rh_pivot_ratio(self._h, _ptr(out)))
        return float(out[0])

    def stage_times(self):
        out = np.zeros(9, np.float32)
        self._rc(lib().rh_stage_times(self._h, _ptr(out)))
        return out


def build():
    from .build import build as _b
    return _b()
