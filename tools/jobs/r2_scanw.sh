mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
cp paper_2101_06550_b200/libpentab.so /tmp/orig.so
for v in orig W4 W2; do
 if [ $v != orig ]; then cp tools/variants/v_$v.so paper_2101_06550_b200/libpentab.so; fi
 echo "== $v"
 timeout 200 python tools/fs_time.py f64 8192:8192 4096:4096 16384:4096 2>&1 | grep -v Warn
 timeout 200 python tools/fs_time.py f32 8192:8192 2>&1 | grep -v Warn
done > gpurun_out/scanw.txt 2>&1
cp /tmp/orig.so paper_2101_06550_b200/libpentab.so
