mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
for i in 1 2; do timeout 300 python bench.py --no-adi --no-sweep --no-ch1d --no-dist --no-cpu --steps 10 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"; done > gpurun_out/e2e.txt 2>&1
