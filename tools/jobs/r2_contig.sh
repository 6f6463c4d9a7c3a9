mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_dist.py tests/test_gpu_stencil_adi.py tests/test_gpu_stress.py tests/test_gpu_cn.py > gpurun_out/contig_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/contig_pytest.log
timeout 600 python bench.py --no-sweep --no-ch1d --no-cpu --steps 10 > gpurun_out/contig_bench.log 2>&1
