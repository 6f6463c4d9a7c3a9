mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_coarsen.py tests/test_gpu_stencil_adi.py tests/test_gpu_dist.py > gpurun_out/cook_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/cook_pytest.log
timeout 600 python bench.py --no-sweep --no-ch1d --no-cpu --no-dist --steps 10 > gpurun_out/cook_bench.log 2>&1
