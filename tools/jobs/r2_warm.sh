mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tp_ --csv python tools/prof_solve.py 8192 f64 6 > gpurun_out/warm_ncu.csv 2>&1
