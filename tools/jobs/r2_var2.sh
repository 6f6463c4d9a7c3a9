mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
cp paper_2101_06550_b200/libpentab.so /tmp/orig.so
for v in orig A B; do
 if [ $v != orig ]; then cp tools/variants/v_$v.so paper_2101_06550_b200/libpentab.so; fi
 echo "== $v"
 timeout 200 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 1024:262144 2>&1 | grep -v Warn
done > gpurun_out/var2.txt 2>&1
cp /tmp/orig.so paper_2101_06550_b200/libpentab.so
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tp_ --csv python tools/prof_solve.py 8192 f64 3 > gpurun_out/var2_ncu.csv 2>&1
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_banded.py tests/test_gpu_dist.py tests/test_gpu_stress.py > gpurun_out/var2_pytest.log 2>&1
tail -3 gpurun_out/var2_pytest.log
