mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_stencil_adi.py tests/test_gpu_dist.py tests/test_gpu_cn.py tests/test_gpu_coarsen.py > gpurun_out/scan8.log 2>&1; echo "rc=$?" >> gpurun_out/scan8.log
timeout 300 python tools/adi_sweep.py 512 >> gpurun_out/scan8.log 2>&1
timeout 300 python tools/fs_time.py f64 8192:8192 512:262144 >> gpurun_out/scan8.log 2>&1
