"""Driver of tools/mb_compute.cu (dev micro-benchmark)."""
import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmbc.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                       "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include"),
                       os.path.join(HERE, "mb_compute.cu"), "-o", SO])
L = ctypes.CDLL(SO)
L.mbc_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.POINTER(ctypes.c_float)]
cyc = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
sink = torch.zeros(148 * 16 * 32 * 7 * 4, dtype=torch.float64, device="cuda")
for store in (0, 1):
    for warps in (1, 4, 8, 12, 16):
        ms = ctypes.c_float()
        items = 200
        L.mbc_run(warps, items, store, cyc.data_ptr(), sink.data_ptr(), ctypes.byref(ms))
        L.mbc_run(warps, items, store, cyc.data_ptr(), sink.data_ptr(), ctypes.byref(ms))
        c = cyc.view(148, 16)[:, :warps].float().mean().item()
        print(f"store={store} warps/SM={warps:2d}: {c / items:8.0f} cycles per warp-item, kernel {ms.value*1e3:8.1f} us, "
              f"tiles/us/SM {warps / 4 * items / (ms.value * 1e3):.3f}", flush=True)
