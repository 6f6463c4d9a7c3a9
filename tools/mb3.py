"""Driver of tools/mb2.cu tile_hold / tma_n (dev micro-benchmark)."""
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
I = ctypes.POINTER(ctypes.c_int)
L.mb2_hold.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_int] * 5 + [F, I]
L.mb2_tma_n.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_int] * 4 + [F]
N = M = 8192
x = torch.rand(N * M, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for ctas in (148, 144, 128, 112):
    ms = ctypes.c_float()
    rc = L.mb2_tma_n(x.data_ptr(), y.data_ptr(), N, M, 16, 256, ctas, 20, ctypes.byref(ms))
    print(f"tma copy W16 R256 ctas={ctas} rc={rc} {ms.value*1e3:8.1f} us {16*N*M/(ms.value*1e-3)/1e9:8.1f} GB/s", flush=True)
for (mr, st, chain, cs) in [(32, 0, 0, 0), (32, 0, 4, 0), (32, 0, 4, 1), (32, 0, 8, 1), (16, 0, 4, 1), (16, 1, 0, 0),
                            (16, 1, 4, 1), (8, 1, 4, 1), (8, 0, 4, 1)]:
    for n in (8192, 4096):
        ms = ctypes.c_float()
        ncl = ctypes.c_int()
        rc = L.mb2_hold(x.data_ptr(), y.data_ptr(), n, M, mr, st, chain, cs, 20, ctypes.byref(ms), ctypes.byref(ncl))
        C = n // (32 * mr)
        print(f"hold N={n} MR={mr} C={C} store_tma={st} chain={chain} csync={cs} clusters={ncl.value} rc={rc} "
              f"{ms.value*1e3:8.1f} us {16*n*M/(ms.value*1e-3)/1e9:8.1f} GB/s", flush=True)
