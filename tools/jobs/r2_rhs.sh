mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_stencil_adi.py tests/test_gpu_coarsen.py tests/test_gpu_dist.py > gpurun_out/rhs_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rhs_pytest.log
timeout 600 python bench.py --no-sweep --no-ch1d --no-dist --no-cpu --steps 20 > gpurun_out/rhs_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_adi_step.py > gpurun_out/rhs_ncu.csv 2>&1
