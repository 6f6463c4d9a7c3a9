set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 120 python tools/fs_time.py f64 64:64 1000:96 2>&1 | tail -3
timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:262144 2>&1 | tail -6
timeout 200 python tools/fs_time.py f32 8192:8192 4096:4096 512:262144 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_ch1d.py -x -q --timeout 300 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_stencil_adi.py tests/test_gpu_dist.py tests/test_gpu_stress.py -x -q --timeout 300 2>&1 | tail -8
timeout 120 python tools/adi_sweep.py 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fc_kernel -s 3 -c 1 -o gpurun_out/fc_prof5 python tools/fs_time.py f64 8192:8192 > gpurun_out/ncu_fc5.log 2>&1; tail -2 gpurun_out/ncu_fc5.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -c 4000 gpurun_out/bench5.json; tail -5 gpurun_out/bench5.err
