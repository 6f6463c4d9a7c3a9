./tools/mb_lat
python -c "import torch; torch.zeros(1).cuda()"
for s in 512:262144 8192:8192; do timeout 100 python tools/fs_time.py f64 $s 2>&1 | tail -12; done
timeout 300 python -m pytest -x -q tests/test_gpu_fused.py 2>&1 | tail -3
