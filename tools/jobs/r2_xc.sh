mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
cp paper_2101_06550_b200/libpentab.so /tmp/orig.so
for v in orig XC; do
 if [ $v != orig ]; then cp tools/variants/v_$v.so paper_2101_06550_b200/libpentab.so; fi
 echo "== $v"
 timeout 300 python tools/adi_sweep.py 512 2>&1 | tail -1
 timeout 300 python bench.py --no-sweep --no-ch1d --no-cpu --no-dist --steps 10 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['cfg3']['us_per_step'], d['ch_adi']['ms_per_step'])"
done > gpurun_out/xc.txt 2>&1
cp /tmp/orig.so paper_2101_06550_b200/libpentab.so
