mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:adi_rhs -s 3 -c 1 -o /tmp/rhs -f python tools/prof_adi_step.py > gpurun_out/ncu_rhs.log 2>&1
ncu -i /tmp/rhs.ncu-rep --page raw --csv > gpurun_out/ncu_rhs.raw.csv 2>/dev/null
ncu -i /tmp/rhs.ncu-rep --page source --csv > gpurun_out/ncu_rhs.src.csv 2>/dev/null
ls -la gpurun_out/ncu_rhs*
