python -c "import torch; torch.zeros(1).cuda()"
timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:262144 2>&1 | tail -6
timeout 200 python tools/fs_time.py f32 8192:8192 512:262144 2>&1 | tail -3
PB_DEV_NOHOLD=1 timeout 100 python tools/fs_time.py f64 8192:8192 512:262144 2>&1 | tail -2
timeout 900 python -m pytest -x -q tests/test_gpu_fused.py tests/test_gpu_stress.py 2>&1 | tail -15
