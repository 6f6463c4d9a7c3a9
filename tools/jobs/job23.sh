python -c "import torch; torch.zeros(1).cuda()"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fh_kernel -s 3 -c 1 -o gpurun_out/fh512b -f python tools/fs_time.py f64 512:262144 > gpurun_out/fh512b.txt 2>&1
