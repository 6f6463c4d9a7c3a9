"""Driver of tools/mb2.cu tma_twophase (dev micro-benchmark)."""
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
L.mb2_twophase.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_int] * 6 + [F]
L.mb2_tma_n.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_int] * 4 + [F]
N = M = 8192
x = torch.rand(N * M, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for ctas in (148, 128, 112, 96, 74):
    ms = ctypes.c_float()
    rc = L.mb2_tma_n(x.data_ptr(), y.data_ptr(), N, M, 16, 256, ctas, 20, ctypes.byref(ms))
    print(f"tma copy W16 R256 ctas={ctas} rc={rc} {ms.value*1e3:8.1f} us {16*N*M/(ms.value*1e-3)/1e9:8.1f} GB/s", flush=True)
cases = []
for W, R in ((16, 256), (16, 128), (32, 128), (32, 64)):
    for G in (8, 16, 32, 64):
        for D in (128, 512, 2048):
            cases.append((W, R, G, D, 148))
cases += [(16, 256, 16, 512, 128), (16, 256, 16, 512, 296), (32, 128, 16, 512, 296), (16, 256, 512, 100000, 148)]
for (W, R, G, D, ctas) in cases:
    ms = ctypes.c_float()
    rc = L.mb2_twophase(x.data_ptr(), y.data_ptr(), N, M, W, R, G, D, ctas, 10, ctypes.byref(ms))
    print(f"twophase W{W} R{R} G{G} D{D} ctas{ctas} rc={rc} {ms.value*1e3:8.1f} us "
          f"{16*N*M/(ms.value*1e-3)/1e9:8.1f} GB/s(alg)", flush=True)
