mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
(timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:512 512:262144;
 timeout 200 python tools/fs_time.py f32 8192:8192 4096:4096 2048:2048 1024:1024 512:262144) > gpurun_out/check.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
