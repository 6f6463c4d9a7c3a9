"""TMA copy bandwidth vs box shape and ring depth on the N = M = 8192 fp64
interleaved array (dev micro-benchmark, driver of tools/mb2.cu)."""
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
N = M = 8192
x = torch.rand(N * M, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for (W, R, S) in [(32, 64, 8), (32, 64, 12), (64, 32, 8), (64, 32, 12), (128, 16, 8), (128, 16, 12), (256, 8, 8),
                  (256, 8, 12), (32, 32, 16), (64, 16, 16), (128, 8, 16), (32, 64, 6), (32, 64, 4)]:
    ms = ctypes.c_float()
    rc = L.mb2_tma(x.data_ptr(), y.data_ptr(), N, M, W, R, S, 1, 0, 10, ctypes.byref(ms))
    print(f"W{W:4d} R{R:3d} S{S:3d} box {W * R * 8 // 1024:3d} KB  in flight {S * W * R * 8 // 1024:4d} KB  rc={rc} "
          f"{ms.value * 1e3:8.1f} us {16 * N * M / (ms.value * 1e-3) / 1e9:8.1f} GB/s", flush=True)
