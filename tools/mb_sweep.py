import ctypes, os, subprocess
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmbs.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                       "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include"), os.path.join(HERE, "mb_sweep.cu"), "-o", SO])
L = ctypes.CDLL(SO)
L.mbs_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
cc = (torch.rand(512 * 8, dtype=torch.float64, device="cuda") * 0.5)
cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
sink = torch.zeros(4, dtype=torch.float64, device="cuda")
for mode in (0, 1, 2):
    ms = ctypes.c_float()
    reps = 1000
    L.mbs_run(mode, cc.data_ptr(), reps, cyc.data_ptr(), sink.data_ptr(), ctypes.byref(ms))
    L.mbs_run(mode, cc.data_ptr(), reps, cyc.data_ptr(), sink.data_ptr(), ctypes.byref(ms))
    c = cyc.float().mean().item()
    print(f"mode {mode}: {c / reps:8.0f} cycles per 32-row sweep ({c / reps / 32:.1f} per row)", flush=True)
