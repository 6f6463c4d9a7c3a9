"""paper_2101_06550_b200 — thin Python binding of libpentab.so (B200, sm_100a).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels (csrc/).  Names follow the C ABI in include/pentab.h.  Buffers
may be torch CUDA tensors (device pointers, enqueued on the current torch
stream unless ``stream`` is given) or numpy arrays (host pointers, staged by
the library).  There is no CPU fallback: if the shared library is missing or
no CUDA device is usable, calls raise.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpentab.so")

PB_OK, PB_EINVAL, PB_EZEROPIVOT, PB_ESINGULAR, PB_ECUDA, PB_ENOMEM, PB_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
PB_F64, PB_F32 = 0, 1
PB_INTERLEAVED, PB_CONTIGUOUS = 0, 1
PB_NONPERIODIC, PB_PERIODIC = 0, 1

# every symbol include/pentab.h declares
EXPORTS = ("pent_factor", "pent_solve", "pent_solve_many", "pent_solve_strided", "pent_solve_info", "pent_refactor", "pent_factor_uniform",
           "pent_destroy", "tri_factor", "tri_solve", "tri_solve_strided", "tri_refactor", "tri_factor_uniform",
           "tri_destroy", "stencil_apply", "ch_workspace_bytes", "ch_adi_step", "ch_adi_step_cook", "ch_free_energy",
           "ch_coarsening_beta", "ch1d_step", "ch_dist_pass_a",
           "ch_dist_pack", "ch_dist_ysweep", "ch_dist_combine", "pb_last_error", "pb_launch_count", "pb_reset_launch_count",
           "pb_device_ok")


class PentabError(RuntimeError):
    def __init__(self, code, msg, sys_idx=-1, row=-1):
        super().__init__(f"pentab error {code}: {msg} (system {sys_idx}, row {row})")
        self.code, self.sys_idx, self.row = code, sys_idx, row


class pb_layout(ctypes.Structure):
    _fields_ = [("n_inner", ctypes.c_int64), ("inner_stride", ctypes.c_int64), ("n_outer", ctypes.c_int64),
                ("outer_stride", ctypes.c_int64), ("row_stride", ctypes.c_int64)]


class pb_grid(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("ny", ctypes.c_int64), ("nx", ctypes.c_int64), ("dtype", ctypes.c_int)]


class pb_window(ctypes.Structure):
    _fields_ = [("left", ctypes.c_int), ("right", ctypes.c_int), ("top", ctypes.c_int), ("bottom", ctypes.c_int)]


class pb_ch_state(ctypes.Structure):
    _fields_ = [("sims", ctypes.c_int64), ("n", ctypes.c_int64), ("dtype", ctypes.c_int),
                ("c_cur", ctypes.c_void_p), ("c_prev", ctypes.c_void_p), ("work", ctypes.c_void_p)]


class pb_ch_params(ctypes.Structure):
    _fields_ = [("D", ctypes.c_double), ("gamma", ctypes.c_double), ("L", ctypes.c_double)]


class pb_ch_noise(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_double), ("seed", ctypes.c_uint64), ("step0", ctypes.c_int64)]


class pb_ch1d_state(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("n", ctypes.c_int64), ("dtype", ctypes.c_int),
                ("c", ctypes.c_void_p), ("work", ctypes.c_void_p)]


class pb_ch1d_params(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("L", ctypes.c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libpentab.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.pent_factor.argtypes = [I64, I64, P, P, P, P, P, I64, I, I, P, ctypes.POINTER(P)]
        L.pent_solve.argtypes = [P, P, I, P]
        L.pent_solve_many.argtypes = [P, P, I, I64, I64, P]
        L.pent_solve_strided.argtypes = [P, P, ctypes.POINTER(pb_layout), P]
        L.tri_solve_strided.argtypes = [P, P, ctypes.POINTER(pb_layout), P]
        L.pent_solve_info.argtypes = [P, I, ctypes.POINTER(ctypes.c_int)]
        L.pent_refactor.argtypes = [P, P, P, P, P, P, P]
        L.pent_factor_uniform.argtypes = [I64, I64, D, D, D, D, D, I, I, P, ctypes.POINTER(P)]
        L.tri_refactor.argtypes = [P, P, P, P, P]
        L.tri_factor_uniform.argtypes = [I64, I64, D, D, D, I, I, P, ctypes.POINTER(P)]
        L.pent_destroy.argtypes = [P]
        L.tri_factor.argtypes = [I64, I64, P, P, P, I64, I, I, P, ctypes.POINTER(P)]
        L.tri_solve.argtypes = [P, P, I, P]
        L.tri_destroy.argtypes = [P]
        L.stencil_apply.argtypes = [ctypes.POINTER(pb_grid), P, P, ctypes.POINTER(pb_window), P, I, P]
        L.ch_workspace_bytes.argtypes = [I64, I64, I, ctypes.POINTER(ctypes.c_size_t)]
        L.ch_adi_step.argtypes = [ctypes.POINTER(pb_ch_state), D, ctypes.POINTER(pb_ch_params), I64, P]
        L.ch1d_step.argtypes = [ctypes.POINTER(pb_ch1d_state), D, ctypes.POINTER(pb_ch1d_params), I64, P]
        L.ch_adi_step_cook.argtypes = [ctypes.POINTER(pb_ch_state), D, ctypes.POINTER(pb_ch_params),
                                       ctypes.POINTER(pb_ch_noise), I64, P]
        L.ch_free_energy.argtypes = [ctypes.POINTER(pb_ch_state), ctypes.POINTER(pb_ch_params), P, P]
        L.ch_coarsening_beta.argtypes = [I64, I64, P, P, P, P]
        L.ch_dist_pass_a.argtypes = [I64, I64, I, P, P, P, D, ctypes.POINTER(pb_ch_params), P]
        L.ch_dist_pack.argtypes = [I64, I64, I64, P, P, P]
        L.ch_dist_ysweep.argtypes = [I64, I64, P, D, ctypes.POINTER(pb_ch_params), P]
        L.ch_dist_combine.argtypes = [I64, I64, I64, I, P, P, P, P]
        L.pb_last_error.argtypes = [ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.c_char_p, ctypes.c_size_t]
        L.pb_launch_count.restype = I64
        L.pb_reset_launch_count.restype = None
        _lib = L
    return _lib


def _check(rc):
    if rc != PB_OK:
        s, r = ctypes.c_int64(-1), ctypes.c_int64(-1)
        buf = ctypes.create_string_buffer(512)
        lib().pb_last_error(ctypes.byref(s), ctypes.byref(r), buf, 512)
        raise PentabError(rc, buf.value.decode(errors="replace"), s.value, r.value)


def _ptr(x):
    """Raw pointer of a torch tensor (device or host) or numpy array (host)."""
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    if hasattr(x, "__array_interface__"):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(x.__array_interface__["data"][0])
    raise TypeError(f"unsupported buffer {type(x)}")


def _stream(x, stream):
    if stream is not None:
        return ctypes.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
    if hasattr(x, "is_cuda") and x.is_cuda:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    return ctypes.c_void_p(0)


def _dtype_code(x):
    name = str(getattr(x, "dtype", ""))
    if name.endswith("float64"):
        return PB_F64
    if name.endswith("float32"):
        return PB_F32
    raise TypeError(f"dtype {name} not supported (float64 / float32)")


def _layout(layout):
    return {"interleaved": PB_INTERLEAVED, "contiguous": PB_CONTIGUOUS, PB_INTERLEAVED: PB_INTERLEAVED,
            PB_CONTIGUOUS: PB_CONTIGUOUS}[layout]


class _Banded:
    _destroy = None
    _strided = None

    def solve_strided(self, rhs, *, n_inner, inner_stride, n_outer=1, outer_stride=0, row_stride, offset=0,
                      stream=None):
        """pent_solve_strided / tri_solve_strided (pentab.h): systems at
        rhs[offset + b*outer_stride + s*inner_stride + i*row_stride], in place."""
        lay = pb_layout(n_inner, inner_stride, n_outer, outer_stride, row_stride)
        base = _ptr(rhs).value + offset * (8 if self.dtype == PB_F64 else 4)
        _check(getattr(lib(), self._strided)(self._h, ctypes.c_void_p(base), ctypes.byref(lay), _stream(rhs, stream)))
        return rhs

    def __init__(self, h, batch, n, dtype):
        self._h, self.batch, self.n, self.dtype = h, batch, n, dtype

    def close(self):
        if self._h:
            getattr(lib(), self._destroy)(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PentaHandle(_Banded):
    _destroy = "pent_destroy"
    _strided = "pent_solve_strided"

    def solve(self, rhs, layout="interleaved", stream=None):
        """pent_solve: in place."""
        _check(lib().pent_solve(self._h, _ptr(rhs), _layout(layout), _stream(rhs, stream)))
        return rhs

    def solve_info(self, layout="interleaved"):
        """pent_solve_info: (cluster size, chunks per CTA, clusters, kernel) of the
        fused solve; kernel 2 = tiles held on chip (one HBM pass), 1 = two-pass
        cluster kernel, 0 = global-scan kernel; all -1 = no fused plan."""
        w = (ctypes.c_int * 4)()
        _check(lib().pent_solve_info(self._h, _layout(layout), w))
        return tuple(w)

    def refactor(self, a, b, c, d, e, stream=None):
        """pent_refactor: new per-system diagonals (device fp64), in place, no sync."""
        _check(lib().pent_refactor(self._h, _ptr(a), _ptr(b), _ptr(c), _ptr(d), _ptr(e), _stream(a, stream)))

    def solve_many(self, rhs, count, batch_stride, layout="interleaved", stream=None):
        _check(lib().pent_solve_many(self._h, _ptr(rhs), _layout(layout), count, batch_stride, _stream(rhs, stream)))
        return rhs


class TriHandle(_Banded):
    _destroy = "tri_destroy"
    _strided = "tri_solve_strided"

    def refactor(self, a, b, c, stream=None):
        """tri_refactor: new per-system diagonals (device fp64), in place, no sync."""
        _check(lib().tri_refactor(self._h, _ptr(a), _ptr(b), _ptr(c), _stream(a, stream)))

    def solve(self, rhs, layout="interleaved", stream=None):
        _check(lib().tri_solve(self._h, _ptr(rhs), _layout(layout), _stream(rhs, stream)))
        return rhs


def _dt(dtype):
    return {"f64": PB_F64, "float64": PB_F64, PB_F64: PB_F64, "f32": PB_F32, "float32": PB_F32, PB_F32: PB_F32}[dtype]


def pent_factor(a, b, c, d, e, *, batch, n, lhs_count=1, periodic=False, dtype="f64", stream=None) -> PentaHandle:
    """Factor once (periodic: Navon P:1498-1620).  a..e: fp64
    buffers of lhs_count*n values, interleaved [i*lhs_count + s]."""
    h = ctypes.c_void_p()
    _check(lib().pent_factor(batch, n, _ptr(a), _ptr(b), _ptr(c), _ptr(d), _ptr(e), lhs_count, int(bool(periodic)),
                             _dt(dtype), _stream(a, stream), ctypes.byref(h)))
    return PentaHandle(h, batch, n, _dt(dtype))


def pent_factor_uniform(a, b, c, d, e, *, batch, n, periodic=False, dtype="f64", stream=None) -> PentaHandle:
    """Shared LHS with constant diagonals (cuPentUniformBatch)."""
    h = ctypes.c_void_p()
    s = ctypes.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream) if stream is not None else \
        ctypes.c_void_p(0)
    _check(lib().pent_factor_uniform(batch, n, a, b, c, d, e, int(bool(periodic)), _dt(dtype), s, ctypes.byref(h)))
    return PentaHandle(h, batch, n, _dt(dtype))


def tri_factor_uniform(a, b, c, *, batch, n, periodic=False, dtype="f64", stream=None) -> TriHandle:
    """Shared tridiagonal LHS with constant diagonals (e.g. CN diffusion)."""
    h = ctypes.c_void_p()
    s = ctypes.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream) if stream is not None else \
        ctypes.c_void_p(0)
    _check(lib().tri_factor_uniform(batch, n, a, b, c, int(bool(periodic)), _dt(dtype), s, ctypes.byref(h)))
    return TriHandle(h, batch, n, _dt(dtype))


def tri_factor(a, b, c, *, batch, n, lhs_count=1, periodic=False, dtype="f64", stream=None) -> TriHandle:
    """Thomas prefactorisation; periodic: Sherman–Morrison."""
    h = ctypes.c_void_p()
    _check(lib().tri_factor(batch, n, _ptr(a), _ptr(b), _ptr(c), lhs_count, int(bool(periodic)), _dt(dtype),
                            _stream(a, stream), ctypes.byref(h)))
    return TriHandle(h, batch, n, _dt(dtype))


def stencil_apply(inp, out, weights, *, left, right, top, bottom, periodic=True, stream=None):
    """cuSten-style window sum.  inp/out: (batch, ny, nx) or (ny, nx)."""
    import numpy as np
    shape = tuple(inp.shape)
    ny, nx = shape[-2], shape[-1]
    batch = 1
    for s in shape[:-2]:
        batch *= s
    g = pb_grid(batch, ny, nx, _dtype_code(inp))
    w = pb_window(left, right, top, bottom)
    wt = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
    _check(lib().stencil_apply(ctypes.byref(g), _ptr(inp), _ptr(out), ctypes.byref(w), _ptr(wt),
                               PB_PERIODIC if periodic else PB_NONPERIODIC, _stream(inp, stream)))
    return out


def ch_workspace_bytes(sims, n, dtype="f64"):
    nb = ctypes.c_size_t()
    _check(lib().ch_workspace_bytes(sims, n, _dt(dtype), ctypes.byref(nb)))
    return nb.value


class CHState:
    """Two time levels + workspace of the ADI CH scheme (device tensors)."""

    def __init__(self, c0, work=None):
        import torch
        assert c0.is_cuda and c0.dim() == 3 and c0.shape[1] == c0.shape[2]
        self.sims, self.n = c0.shape[0], c0.shape[1]
        self.dtype = _dtype_code(c0)
        self.bufs = [c0.clone().contiguous(), c0.clone().contiguous()]  # C^n, C^{n-1}
        nb = ch_workspace_bytes(self.sims, self.n, self.dtype)
        self.work = work if work is not None else torch.empty(max(nb, 8), dtype=torch.uint8, device=c0.device)
        self.state = pb_ch_state(self.sims, self.n, self.dtype, self.bufs[0].data_ptr(), self.bufs[1].data_ptr(),
                                 self.work.data_ptr())

    def _tensor(self, ptr):
        return self.bufs[0] if self.bufs[0].data_ptr() == ptr else self.bufs[1]

    @property
    def c_cur(self):
        return self._tensor(self.state.c_cur)

    @property
    def c_prev(self):
        return self._tensor(self.state.c_prev)


def ch_adi_step(state: CHState, dt, *, D=1.0, gamma=0.01, L, nsteps=1, stream=None):
    """nsteps of Eq 3.1 on device; levels rotate in `state`."""
    p = pb_ch_params(D, gamma, L)
    _check(lib().ch_adi_step(ctypes.byref(state.state), dt, ctypes.byref(p), nsteps, _stream(state.bufs[0], stream)))
    return state


def ch_adi_step_cook(state: CHState, dt, *, sigma, seed, step0=0, D=1.0, gamma=0.01, L, nsteps=1, stream=None):
    """nsteps of the Cahn–Hilliard–Cook equation on device."""
    p = pb_ch_params(D, gamma, L)
    nz = pb_ch_noise(sigma, seed, step0)
    _check(lib().ch_adi_step_cook(ctypes.byref(state.state), dt, ctypes.byref(p), ctypes.byref(nz), nsteps,
                                  _stream(state.bufs[0], stream)))
    return state


def ch_free_energy(state: CHState, F, *, gamma=0.01, L, stream=None):
    """F (reading r24) of every simulation into the device tensor F."""
    p = pb_ch_params(1.0, gamma, L)
    _check(lib().ch_free_energy(ctypes.byref(state.state), ctypes.byref(p), _ptr(F), _stream(state.bufs[0], stream)))
    return F


def ch_coarsening_beta(t, F, beta, stream=None):
    """beta = -(t/F) dF/dt (reading r27); t [nt], F and beta [nt][sims], device."""
    nt = t.shape[0]
    _check(lib().ch_coarsening_beta(nt, F.numel() // nt, _ptr(t), _ptr(F), _ptr(beta), _stream(F, stream)))
    return beta


class CH1DState:
    """A batch of 1D CH systems (thesis §6.2): interleaved [n][batch] level +
    a same-sized work buffer (device tensors); the two swap every step."""

    def __init__(self, c0):
        import torch
        assert c0.is_cuda and c0.dim() == 2, "c0: (n, batch) device tensor, system fastest"
        self.n, self.batch = c0.shape
        self.dtype = _dtype_code(c0)
        self.bufs = [c0.clone().contiguous(), torch.empty_like(c0)]
        self.state = pb_ch1d_state(self.batch, self.n, self.dtype, self.bufs[0].data_ptr(), self.bufs[1].data_ptr())

    @property
    def c(self):
        return self.bufs[0] if self.bufs[0].data_ptr() == self.state.c else self.bufs[1]


def ch1d_step(state: CH1DState, dt, *, gamma=0.01, L, nsteps=1, stream=None):
    """nsteps of eq6:1Dnumerical on device; levels swap in `state`."""
    p = pb_ch1d_params(gamma, L)
    _check(lib().ch1d_step(ctypes.byref(state.state), dt, ctypes.byref(p), nsteps, _stream(state.bufs[0], stream)))
    return state


def launch_count() -> int:
    return int(lib().pb_launch_count())


def reset_launch_count():
    lib().pb_reset_launch_count()


def device_ok() -> bool:
    return lib().pb_device_ok() == PB_OK


# ---------------------------------------------------------------- row-partitioned ADI (configs[4])
def ch_dist_pass_a(cn_ext, cm_ext, w, *, rows, n, dt, D=1.0, gamma=0.01, L, stream=None):
    """RHS + x-sweep of a row block with 2 halo rows each side (pentab.h)."""
    p = pb_ch_params(D, gamma, L)
    _check(lib().ch_dist_pass_a(rows, n, _dtype_code(cn_ext), _ptr(cn_ext), _ptr(cm_ext), _ptr(w), dt, ctypes.byref(p),
                                _stream(w, stream)))


def ch_dist_pack(w, packed, *, rows, n, parts, stream=None):
    _check(lib().ch_dist_pack(rows, n, parts, _ptr(w), _ptr(packed), _stream(w, stream)))


def ch_dist_ysweep(cols, *, ncols, n, dt, D=1.0, gamma=0.01, L, stream=None):
    """y-sweep of the rank's [n][ncols] column block, in place (pentab.h)."""
    p = pb_ch_params(D, gamma, L)
    _check(lib().ch_dist_ysweep(ncols, n, _ptr(cols), dt, ctypes.byref(p), _stream(cols, stream)))


def ch_dist_combine(cn_ext, cm_ext, v_packed, *, rows, n, parts, stream=None):
    _check(lib().ch_dist_combine(rows, n, parts, _dtype_code(cn_ext), _ptr(cn_ext), _ptr(cm_ext), _ptr(v_packed),
                                 _stream(cn_ext, stream)))
