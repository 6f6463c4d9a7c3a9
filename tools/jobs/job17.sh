python -c "import torch; torch.zeros(1).cuda()"
for d in 0 253; do
PB_DEV_DBG=$d timeout 300 ncu --set full --clock-control none -k regex:fc_kernel -s 3 -c 1 -o gpurun_out/fc_dbg$d -f python tools/fs_time.py f64 8192:8192 > gpurun_out/fc_dbg$d.txt 2>&1
done
