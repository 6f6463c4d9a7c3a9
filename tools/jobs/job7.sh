python -c "import torch; torch.zeros(1).cuda()"
for cs in 0 8 16 4; do for d in 0 1 2 3; do echo "CS=$cs DBG=$d"; PB_DEV_CS=$cs PB_DEV_DBG=$d timeout 100 python tools/fs_time.py f64 8192:8192 4096:4096 512:262144 2>&1 | tail -3; done; done
