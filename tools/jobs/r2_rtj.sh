mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
cp paper_2101_06550_b200/libpentab.so /tmp/orig.so
for v in orig B21 B42 B8J8; do
 if [ $v != orig ]; then cp tools/variants/v_$v.so paper_2101_06550_b200/libpentab.so; fi
 echo "== $v"
 timeout 300 python tools/adi_sweep.py 512 2>&1 | tail -1
 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:adi_rhs python tools/prof_adi_step.py 2>&1 | grep gpu__time | tail -1 | awk -F'","' '{print $NF}'
done > gpurun_out/rtj.txt 2>&1
cp /tmp/orig.so paper_2101_06550_b200/libpentab.so
