python -c "import torch; torch.zeros(1).cuda()"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fh_kernel -s 3 -c 1 -o gpurun_out/fh512 -f python tools/fs_time.py f64 512:262144 > gpurun_out/fh512.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fh_kernel -s 3 -c 1 -o gpurun_out/fh8192 -f python tools/fs_time.py f64 8192:8192 > gpurun_out/fh8192.txt 2>&1
