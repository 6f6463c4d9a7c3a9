mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 ncu --set full --clock-control none --import-source on -s 18 -c 6 -o /tmp/r02c_adi -f python tools/prof_adi_step.py > gpurun_out/r02c_adi.log 2>&1
ncu -i /tmp/r02c_adi.ncu-rep --page raw --csv > gpurun_out/r02c_adi.raw.csv 2>/dev/null
