mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_stencil_adi.py tests/test_gpu_coarsen.py tests/test_gpu_dist.py tests/test_gpu_stress.py > gpurun_out/adiy_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/adiy_pytest.log
timeout 300 python tools/adi_sweep.py 512 > gpurun_out/adiy.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_adi_step.py > gpurun_out/adiy_ncu.csv 2>&1
