mkdir -p gpurun_out
PB_EXTRA_NVCC_FLAGS=-DFH_PROF python -c "from paper_2101_06550_b200 import build as b; b.build(force=True)" > gpurun_out/fhprof_build.txt 2>&1
python -c "import torch; torch.zeros(1).cuda()"
for s in 512:262144 8192:8192 2048:2048; do
timeout 200 python tools/fs_time.py f64 $s
done > gpurun_out/fhprof.txt 2>&1
nvidia-smi -q | grep -i -A3 "clocks" | head -20 >> gpurun_out/fhprof.txt
