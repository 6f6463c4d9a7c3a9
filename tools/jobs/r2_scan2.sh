mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
(timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 16384:4096 20000:2048;
 timeout 200 python tools/fs_time.py f32 8192:8192 16384:4096) > gpurun_out/scan2.txt 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_dist.py tests/test_gpu_stress.py > gpurun_out/scan2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/scan2_pytest.log
timeout 600 python bench.py --no-sweep --no-ch1d --no-cpu --no-adi --steps 10 > gpurun_out/scan2_bench.log 2>&1
