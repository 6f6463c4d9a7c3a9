mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
for p in 0 1 2; do
echo "== PATH $p" 
PB_DEV_PATH=$p timeout 200 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 512:262144 2>&1 | grep -v Warn
PB_DEV_PATH=$p timeout 200 python tools/fs_time.py f32 8192:8192 512:262144 2>&1 | grep -v Warn
done > gpurun_out/paths.txt
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py -k "16384 or cluster_and_global" > gpurun_out/pt_fix.log 2>&1
tail -3 gpurun_out/pt_fix.log
