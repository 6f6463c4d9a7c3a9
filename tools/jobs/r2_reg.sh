mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 600 python bench.py --no-adi --no-ch1d --no-cpu --no-dist --steps 10 > gpurun_out/reg_bench.log 2>&1; echo "rc=$?" >> gpurun_out/reg_bench.log
