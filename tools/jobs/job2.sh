set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 300 python tools/fs_time.py f64 64:64 8:4 1000:96 2>&1 | tail -5
timeout 600 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:262144 2>&1 | tail -8
timeout 600 python tools/fs_time.py f32 8192:8192 4096:4096 512:262144 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_banded.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_stencil_adi.py tests/test_gpu_dist.py -x -q 2>&1 | tail -15
timeout 300 python tools/adi_sweep.py 2>&1 | tail -2
