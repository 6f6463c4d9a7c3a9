python -c "import torch; torch.zeros(1).cuda()"
timeout 150 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:262144 2>&1 | tail -5
timeout 100 python tools/fs_time.py f32 8192:8192 4096:4096 512:262144 2>&1 | tail -3
timeout 120 python tools/adi_sweep.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_ch1d.py tests/test_gpu_cn.py -x -q --timeout 300 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_stencil_adi.py tests/test_gpu_dist.py tests/test_gpu_stress.py -x -q --timeout 300 2>&1 | tail -4
