mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
cp paper_2101_06550_b200/libpentab.so /tmp/orig.so
for v in orig IA; do
 if [ $v != orig ]; then cp tools/variants/v_$v.so paper_2101_06550_b200/libpentab.so; fi
 echo "== $v"
 timeout 300 python tools/adi_sweep.py 512 2>&1 | tail -1
 timeout 300 python tools/fs_time.py f64 512:262144 512:65536 2>&1 | grep -v Warn
done > gpurun_out/ia.txt 2>&1
cp /tmp/orig.so paper_2101_06550_b200/libpentab.so
