mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py -k "host" tests/test_gpu_banded.py -k "host" > gpurun_out/e2e2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e2e2_pytest.log
for i in 1 2 3; do timeout 300 python bench.py --no-adi --no-sweep --no-ch1d --no-dist --no-cpu --steps 10 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"; done > gpurun_out/e2e2.txt 2>&1
