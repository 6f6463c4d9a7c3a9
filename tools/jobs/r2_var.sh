mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
cp paper_2101_06550_b200/libpentab.so /tmp/orig.so
for v in A B C D E; do
 cp tools/variants/v_$v.so paper_2101_06550_b200/libpentab.so
 echo "== $v"
 timeout 200 python tools/fs_time.py f64 8192:8192 4096:4096 2048:2048 2>&1 | grep -v Warn
done > gpurun_out/var.txt 2>&1
cp /tmp/orig.so paper_2101_06550_b200/libpentab.so
