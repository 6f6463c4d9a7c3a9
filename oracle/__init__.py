"""CPU ORACLE for the hot path of arxiv/paper_2101_06550 (Gloster thesis).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with the CUDA product path
(``paper_2101_06550_b200``) and neither side imports the other; the only
shared module is ``synth`` (seeded input generators, no method arithmetic).

The arithmetic lives in ``oracle/oracle.c`` (plain scalar fp64 C, the paper's
algorithms step by step, each citing PAPER.md lines); this module is a thin
ctypes/numpy wrapper plus the paper's error metrics.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
against dense LU, closed forms (circulant eigenvalues, FFT), invariants (mass,
fixed points) and the printed Tables 3.1 and 6.1 — see DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, EZEROPIVOT, ESINGULAR = 0, -1, -2, -3


class OracleError(RuntimeError):
    def __init__(self, code, sys_idx=-1, row=-1):
        super().__init__(f"oracle error {code} (system {sys_idx}, row {row})")
        self.code, self.sys_idx, self.row = code, sys_idx, row


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain -O2, no intrinsics, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        Ci = ctypes.c_int
        L.orc_penta_factor.argtypes = [I64] + [P] * 10 + [P]
        L.orc_penta_solve.argtypes = [I64] + [P] * 7
        L.orc_penta_solve.restype = None
        L.orc_penta_batch_solve.argtypes = [I64, I64, Ci, I64, Ci] + [P] * 7 + [P, P]
        L.orc_tri_factor.argtypes = [I64, P, P, P, P, P]
        L.orc_tri_solve.argtypes = [I64, P, P, P, P, P]
        L.orc_tri_solve.restype = None
        L.orc_tri_batch_solve.argtypes = [I64, I64, Ci, I64, Ci] + [P] * 5 + [P, P]
        L.orc_stencil_apply.argtypes = [I64, I64, I64, Ci, Ci, Ci, Ci, P, Ci, P, P]
        L.orc_ch_rhs.argtypes = [I64, I64, D, D, D, D, P, P, P]
        L.orc_ch_adi_steps.argtypes = [I64, I64, D, D, D, D, I64, P, P]
        L.orc_ch1d_steps.argtypes = [I64, I64, D, D, D, I64, P]
        U64 = ctypes.c_uint64
        L.orc_ch_free_energy.argtypes = [I64, I64, D, D, P, P]
        L.orc_coarsening_beta.argtypes = [I64, I64, P, P, P]
        L.orc_cook_rho.argtypes = [U64, I64, I64, I64, P, P]
        L.orc_cook_rho.restype = None
        L.orc_cook_noise.argtypes = [I64, I64, D, D, D, U64, I64, P]
        L.orc_ch_adi_steps_cook.argtypes = [I64, I64, D, D, D, D, D, U64, I64, I64, P, P]
        _lib = L
    return _lib


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _p(x):
    return x.ctypes.data_as(ctypes.c_void_p)


def _check(rc, bad_sys=None, bad_row=None):
    if rc != 0:
        raise OracleError(rc, -1 if bad_sys is None else bad_sys.value, -1 if bad_row is None else bad_row.value)


# ----------------------------------------------------------------- penta
def penta_factor(a, b, c, d, e):
    """14-step LR factorisation. Returns (alpha, beta, gamma, delta, eps)."""
    a, b, c, d, e = map(_f64, (a, b, c, d, e))
    n = c.shape[0]
    outs = [np.zeros(n) for _ in range(5)]
    row = ctypes.c_int64(-1)
    rc = lib().orc_penta_factor(n, _p(a), _p(b), _p(c), _p(d), _p(e), *map(_p, outs), ctypes.byref(row))
    _check(rc, None, row)
    return tuple(outs)


def penta_solve_factored(fac, f):
    """Forward g and back substitution x."""
    fac = [_f64(v) for v in fac]
    f = _f64(f)
    x = np.zeros_like(f)
    lib().orc_penta_solve(f.shape[0], *map(_p, fac), _p(f), _p(x))
    return x


def penta_batch_solve(a, b, c, d, e, rhs, *, n, m, layout="interleaved", periodic=False):
    """Batched solve.  rhs flat of n*m (interleaved i*m+s or contiguous s*n+i).
    a..e flat of n*lhs_count, interleaved [i*lhs_count + s] (lhs_count = 1 or m)."""
    a, b, c, d, e = map(_f64, (a, b, c, d, e))
    rhs = _f64(rhs).reshape(-1)
    lhs_count = a.size // n
    x = np.zeros_like(rhs)
    bs, br = ctypes.c_int64(-1), ctypes.c_int64(-1)
    lay = 0 if layout == "interleaved" else 1
    rc = lib().orc_penta_batch_solve(n, m, lay, lhs_count, int(periodic), _p(a), _p(b), _p(c), _p(d), _p(e),
                                     _p(rhs), _p(x), ctypes.byref(bs), ctypes.byref(br))
    _check(rc, bs, br)
    return x


# ----------------------------------------------------------------- tri
def tri_factor(a, b, c):
    """Thomas pre-factorisation chat."""
    a, b, c = map(_f64, (a, b, c))
    n = b.shape[0]
    ch = np.zeros(n)
    row = ctypes.c_int64(-1)
    rc = lib().orc_tri_factor(n, _p(a), _p(b), _p(c), _p(ch), ctypes.byref(row))
    _check(rc, None, row)
    return ch


def tri_solve_factored(a, b, chat, d):
    a, b, chat, d = map(_f64, (a, b, chat, d))
    x = np.zeros_like(d)
    lib().orc_tri_solve(d.shape[0], _p(a), _p(b), _p(chat), _p(d), _p(x))
    return x


def tri_batch_solve(a, b, c, rhs, *, n, m, layout="interleaved", periodic=False):
    a, b, c = map(_f64, (a, b, c))
    rhs = _f64(rhs).reshape(-1)
    lhs_count = a.size // n
    x = np.zeros_like(rhs)
    bs, br = ctypes.c_int64(-1), ctypes.c_int64(-1)
    lay = 0 if layout == "interleaved" else 1
    rc = lib().orc_tri_batch_solve(n, m, lay, lhs_count, int(periodic), _p(a), _p(b), _p(c), _p(rhs), _p(x),
                                   ctypes.byref(bs), ctypes.byref(br))
    _check(rc, bs, br)
    return x


# ----------------------------------------------------------------- stencil
def stencil_apply(grid, weights, *, left, right, top, bottom, periodic=True, out=None):
    """cuSten-style window sum.  grid: (batch, ny, nx) or (ny, nx)."""
    g = _f64(grid)
    shape = g.shape
    g3 = g.reshape((-1,) + shape[-2:])
    w = _f64(weights).reshape(-1)
    assert w.size == (top + bottom + 1) * (left + right + 1)
    o = np.zeros_like(g3) if out is None else _f64(out).reshape(g3.shape).copy()
    rc = lib().orc_stencil_apply(g3.shape[0], g3.shape[1], g3.shape[2], left, right, top, bottom, _p(w),
                                 int(periodic), _p(g3), _p(o))
    _check(rc)
    return o.reshape(shape)


# ----------------------------------------------------------------- CH
def ch_rhs(cn, cm, *, dt, D, gamma, L):
    cn, cm = _f64(cn), _f64(cm)
    shape = cn.shape
    n = shape[-1]
    sims = cn.size // (n * n)
    R = np.zeros_like(cn)
    rc = lib().orc_ch_rhs(sims, n, dt, D, gamma, L, _p(cn), _p(cm), _p(R))
    _check(rc)
    return R


def ch_adi_steps(cn, cm, nsteps, *, dt, D, gamma, L):
    """Advance Eq 3.1 nsteps; returns (C^n, C^{n-1}) after the steps (copies)."""
    cn, cm = _f64(cn).copy(), _f64(cm).copy()
    n = cn.shape[-1]
    sims = cn.size // (n * n)
    rc = lib().orc_ch_adi_steps(sims, n, dt, D, gamma, L, nsteps, _p(cn), _p(cm))
    _check(rc)
    return cn, cm


def ch1d_steps(c, nsteps, *, n, m, dt, gamma, L):
    """1D semi-implicit CH, batch interleaved c[i*m+s]."""
    c = _f64(c).reshape(-1).copy()
    rc = lib().orc_ch1d_steps(n, m, dt, gamma, L, nsteps, _p(c))
    _check(rc)
    return c


# ----------------------------------------------------------------- coarsening statistics
def ch_free_energy(c, *, L, gamma):
    """F of P:819-825 per simulation (reading r24: periodic forward differences)."""
    c = _f64(c)
    n = c.shape[-1]
    sims = c.size // (n * n)
    F = np.zeros(sims)
    _check(lib().orc_ch_free_energy(sims, n, L, gamma, _p(c), _p(F)))
    return F


def coarsening_beta(t, F):
    """beta = -(t/F) dF/dt from samples F[k][sim] at times t[k] (reading r27)."""
    t, F = _f64(t), _f64(F)
    nt = t.shape[0]
    F2 = F.reshape(nt, -1)
    beta = np.zeros_like(F2)
    _check(lib().orc_coarsening_beta(nt, F2.shape[1], _p(t), _p(F2), _p(beta)))
    return beta.reshape(F.shape)


def cook_rho(seed, step, sim, cell):
    """The counter-based N(0,1) pair (rho_x, rho_y) of one cell (reading r26)."""
    rx, ry = np.zeros(1), np.zeros(1)
    lib().orc_cook_rho(seed, step, sim, cell, _p(rx), _p(ry))
    return float(rx[0]), float(ry[0])


def cook_noise(sims, n, *, dt, L, sigma, seed, step):
    """eta = sqrt(sigma/(dx^2 dt)) div rho, central differences (r26)."""
    eta = np.zeros((sims, n, n))
    _check(lib().orc_cook_noise(sims, n, dt, L, sigma, seed, step, _p(eta)))
    return eta


def ch_adi_steps_cook(cn, cm, nsteps, *, dt, D, gamma, L, sigma, seed, step0=0):
    """Eq 3.1 with the Cahn–Hilliard–Cook noise + 2/3 dt eta^n in the RHS (r25)."""
    cn, cm = _f64(cn).copy(), _f64(cm).copy()
    n = cn.shape[-1]
    sims = cn.size // (n * n)
    _check(lib().orc_ch_adi_steps_cook(sims, n, dt, D, gamma, L, sigma, seed, step0, nsteps, _p(cn), _p(cm)))
    return cn, cm


# ----------------------------------------------------------------- error metrics
def convergence_error_2d(fine, coarse, L):
    """E_N of eq2:converge2D: the 4-point average of fine cells
    (2i-1,2j-1),(2i-1,2j),(2i,2j-1),(2i,2j) against coarse (i,j), times
    dx_{N/2}^2, over Omega = L^2."""
    fine, coarse = _f64(fine), _f64(coarse)
    nc = coarse.shape[-1]
    avg = (fine[0::2, 0::2] + fine[1::2, 0::2] + fine[0::2, 1::2] + fine[1::2, 1::2]) / 4.0
    dxc = L / nc
    return float(np.sum(np.abs(avg - coarse)) * dxc * dxc / (L * L))


def convergence_error_1d(fine, coarse, L):
    """E_N of eq2:converge1D: sum |F(x_{2i-1}) - C(x_i)| dx_{N/2} / Omega."""
    fine, coarse = _f64(fine), _f64(coarse)
    nc = coarse.shape[-1]
    return float(np.sum(np.abs(fine[0::2] - coarse)) * (L / nc) / L)


def l2_error(num, exact):
    """epsilon_N of eq:myerr."""
    num, exact = _f64(num), _f64(exact)
    return float(np.sqrt(np.mean((num - exact) ** 2)))
