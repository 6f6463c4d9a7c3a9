mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
(timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:262144;
 timeout 200 python tools/fs_time.py f32 8192:8192 4096:4096 2048:2048;
 PB_DEV_PATH=3 timeout 200 python tools/fs_time.py f64 512:262144) > gpurun_out/tp1.txt 2>&1
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_stress.py > gpurun_out/tp1_pytest.log 2>&1
tail -30 gpurun_out/tp1_pytest.log
./tools/mb_lat > gpurun_out/mb_lat.txt 2>&1
