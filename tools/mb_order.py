"""TMA copy bandwidth vs tile ORDER (DRAM page locality) on the N = M = 8192
fp64 interleaved array: order 0 = row-block-major (concurrent CTAs read
adjacent 256-byte column bands of the same rows), order 1 = group-major
(concurrent CTAs read different row blocks of one column band)."""
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
for (N, M) in [(8192, 8192), (512, 262144)]:
    x = torch.rand(N * M, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for order in (0, 1):
        for (W, R, S) in [(32, 64, 8), (32, 64, 4), (64, 32, 8), (32, 32, 8)]:
            ms = ctypes.c_float()
            rc = L.mb2_tma(x.data_ptr(), y.data_ptr(), N, M, W, R, S, 1, order, 10, ctypes.byref(ms))
            print(f"N{N} M{M} order {order} W{W:4d} R{R:3d} S{S:3d} rc={rc} "
                  f"{ms.value * 1e3:8.1f} us {16 * N * M / (ms.value * 1e-3) / 1e9:8.1f} GB/s", flush=True)
