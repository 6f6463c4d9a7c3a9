mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
python -c "import torch; torch.zeros(1).cuda()"
timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:262144 > gpurun_out/fs_f64.txt 2>&1
timeout 300 python tools/fs_time.py f32 8192:8192 4096:4096 512:262144 > gpurun_out/fs_f32.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --adi-steps 5 --no-cpu > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
