set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/ring_stress.sh 5 2>&1 | tee gpurun_out/r2_ring_stress.txt
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2_gputest1.txt
timeout 600 python bench.py --steps 50 --warmup 5 --cpu-budget 2 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
