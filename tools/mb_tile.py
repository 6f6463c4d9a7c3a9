"""Driver of tools/mb_tile.cu (dev micro-benchmark)."""
import ctypes
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmb.so")
if True:
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", os.path.join(HERE, "mb_tile.cu"), "-o", SO])
L = ctypes.CDLL(SO)
L.mb_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                     ctypes.POINTER(ctypes.c_float)]
NAMES = ["stream_copy", "W16 NT512 MR32", "W16 NT512 MR32 +cluster8 sync", "W16 NT512 MR16", "W16 NT512 MR16 +cluster16",
         "W32 NT512 MR32", "W32 NT512 MR16", "W64 NT512 MR32", "W16 NT256 MR32", "W16 NT256 MR32 +cluster16",
         "W32 NT1024 MR16", "W8 NT256 MR32", "W8 NT256 MR32 +cl", "W4 NT128 MR32", "W4 NT128 MR32 +cl",
         "W8 NT128 MR32", "W8 NT128 MR64 +cl", "W4 NT64 MR64 +cl", "W16 NT256 MR32", "W32 NT256 MR32"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x = torch.rand(n * n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for v, name in enumerate(NAMES):
    ms = ctypes.c_float()
    rc = L.mb_run(v, x.data_ptr(), y.data_ptr(), n, n, 20, ctypes.byref(ms))
    print(f"{v:2d} {name:32s} rc={rc} {ms.value * 1e3:9.1f} us  {2 * 8 * n * n / (ms.value * 1e-3) / 1e9:8.1f} GB/s", flush=True)

out = torch.tensor([1.0000001, 1e-9, 0.5, 0], dtype=torch.float64, device="cuda")
outf = torch.tensor([1.0001, 1e-5, 0.5, 0], dtype=torch.float32, device="cuda")
cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
L.mb_lat.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int]
L.mb_lat(out.data_ptr(), outf.data_ptr(), cyc.data_ptr(), 1000)
print("dfma latency cyc/op", cyc[0].item() / 16000, "ffma", cyc[1].item() / 16000)
