mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
cp tools/variants/v_prof.so paper_2101_06550_b200/libpentab.so
for s in 8192:8192 2048:2048; do timeout 200 python tools/prof_solve.py ${s%%:*} f64 10 2>&1 | tail -2; done > gpurun_out/prof.txt 2>&1
