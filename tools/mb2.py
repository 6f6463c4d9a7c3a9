"""Driver of tools/mb2.cu (dev micro-benchmark)."""
import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmb2.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       os.path.join(HERE, "mb2.cu"), "-o", SO])
L = ctypes.CDLL(SO)
F = ctypes.POINTER(ctypes.c_float)
L.mb2_tma.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_int] * 6 + [F]
L.mb2_ldg_stream.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_int] * 4 + [F]
L.mb2_l2.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, F]

N = M = 8192
x = torch.rand(N * M, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)


def rep(name, rc, ms, nbytes):
    print(f"{name:48s} rc={rc} {ms * 1e3:9.1f} us {nbytes / (ms * 1e-3) / 1e9:8.1f} GB/s", flush=True)


for (W, R, S, cps, order) in [(16, 256, 4, 1, 0), (16, 256, 4, 1, 1), (16, 128, 6, 1, 0), (16, 256, 6, 1, 0),
                              (16, 64, 8, 2, 0), (32, 128, 4, 1, 0), (32, 64, 6, 2, 0), (8, 256, 8, 1, 0),
                              (8, 256, 4, 2, 0), (4, 256, 8, 2, 0), (16, 256, 3, 2, 0), (64, 64, 4, 1, 0),
                              (16, 32, 8, 4, 0)]:
    ms = ctypes.c_float()
    rc = L.mb2_tma(x.data_ptr(), y.data_ptr(), N, M, W, R, S, cps, order, 20, ctypes.byref(ms))
    rep(f"tma W{W} R{R} S{S} cps{cps} order{order}", rc, ms.value, 16 * N * M)
ok = torch.equal(x, y)
print("tma copy exact:", ok)
for (W, RB, nt) in [(16, 1024, 256), (16, 256, 256), (8, 512, 256), (32, 512, 256), (64, 256, 256), (128, 128, 256)]:
    ms = ctypes.c_float()
    rc = L.mb2_ldg_stream(x.data_ptr(), y.data_ptr(), N, M, W, RB, nt, 20, ctypes.byref(ms))
    rep(f"ldg tile stream W{W} RB{RB} nt{nt}", rc, ms.value, 16 * N * M)
for mb in (8, 24, 48, 96):
    n = mb * 1024 * 1024 // 8
    buf = torch.rand(n, dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    ms = ctypes.c_float()
    reps = 20
    rc = L.mb2_l2(buf.data_ptr(), n, reps, out.data_ptr(), ctypes.byref(ms))
    rep(f"l2 read {mb} MB", rc, ms.value, 8 * n * reps)
