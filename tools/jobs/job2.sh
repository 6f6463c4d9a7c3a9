set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 120 python tools/fs_time.py f64 64:64 8:4 1000:96 2>&1 | tail -5
timeout 300 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:1024 512:262144 2>&1 | tail -8
timeout 200 python tools/fs_time.py f32 8192:8192 4096:4096 512:262144 2>&1 | tail -5
for tool in synccheck racecheck memcheck; do
  timeout 300 compute-sanitizer --tool $tool --print-limit 20 python tools/tp_repeat.py 300 96 3 > gpurun_out/fs_sanitizer_$tool.txt 2>&1
  echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/fs_sanitizer_$tool.txt | tail -1)"
done
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_banded.py -x -q --timeout 120 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_ch1d.py -x -q -s --timeout 300 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_stencil_adi.py tests/test_gpu_dist.py tests/test_gpu_stress.py -x -q --timeout 300 2>&1 | tail -15
timeout 120 python tools/adi_sweep.py 2>&1 | tail -2
