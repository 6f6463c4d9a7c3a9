python -c "import torch; torch.zeros(1).cuda()"
for d in 0 1 4 5; do echo "DBG=$d"; PB_DEV_DBG=$d timeout 100 python tools/fs_time.py f64 8192:8192 512:262144 2>&1 | tail -2; done
for cs in 1 2 4 8; do echo "CS=$cs"; PB_DEV_CS=$cs PB_DEV_DBG=5 timeout 100 python tools/fs_time.py f64 8192:8192 2>&1 | tail -1; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fc_kernel -s 3 -c 1 -o gpurun_out/fc_prof11 python tools/fs_time.py f64 512:262144 > /dev/null 2>&1; echo ncu done
