python -c "import torch; torch.zeros(1).cuda()"
for d in 0 8 5 13; do echo "DBG=$d"; PB_DEV_DBG=$d timeout 100 python tools/fs_time.py f64 8192:8192 512:262144 2>&1 | tail -2; done
