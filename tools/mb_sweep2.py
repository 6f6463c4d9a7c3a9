import ctypes, os, subprocess
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmbs2.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                       "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include"), os.path.join(HERE, "mb_sweep2.cu"), "-o", SO])
L = ctypes.CDLL(SO)
L.mbs2_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
sink = torch.zeros(4, dtype=torch.float64, device="cuda")
for thr in (32, 128, 256, 512):
    ms = ctypes.c_float()
    reps = 500
    L.mbs2_run(thr, reps, cyc.data_ptr(), sink.data_ptr(), ctypes.byref(ms))
    L.mbs2_run(thr, reps, cyc.data_ptr(), sink.data_ptr(), ctypes.byref(ms))
    c = cyc.float().mean().item()
    print(f"{thr // 32:2d} warps/SM: {c / reps / 32:6.1f} cycles per row per warp", flush=True)
