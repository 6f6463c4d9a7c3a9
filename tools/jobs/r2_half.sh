mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
(timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 1024:262144;
 timeout 200 python tools/fs_time.py f32 8192:8192 4096:4096 2048:2048) > gpurun_out/half.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tp_ --csv python tools/prof_solve.py 8192 f64 3 > gpurun_out/half_ncu.csv 2>&1
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_cn.py > gpurun_out/half_pytest.log 2>&1
tail -3 gpurun_out/half_pytest.log
