mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
