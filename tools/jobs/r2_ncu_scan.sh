mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tp_scan -s 2 -c 1 -o /tmp/scan -f python tools/prof_solve.py 8192 f64 4 > gpurun_out/ncu_scan.log 2>&1
ncu -i /tmp/scan.ncu-rep --page raw --csv > gpurun_out/ncu_scan.raw.csv 2>/dev/null
ncu -i /tmp/scan.ncu-rep --page source --csv > gpurun_out/ncu_scan.src.csv 2>/dev/null
