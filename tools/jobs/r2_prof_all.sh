mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$t.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$t.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 5 --warmup 3 --adi-steps 5 --no-cpu > gpurun_out/r02_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tp_ -s 6 -c 3 -o gpurun_out/r02_solve -f python tools/prof_solve.py 8192 f64 4 > gpurun_out/r02_solve.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tp_ -s 6 -c 3 -o gpurun_out/r02_solve32 -f python tools/prof_solve.py 8192 f32 4 > gpurun_out/r02_solve32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 12 -c 4 -o gpurun_out/r02_adi -f python tools/prof_adi_step.py > gpurun_out/r02_adi.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fh_ -s 2 -c 1 -o gpurun_out/r02_ch1d -f python tools/prof_ch1d.py > gpurun_out/r02_ch1d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil -c 1 -o gpurun_out/r02_stencil -f python tools/prof_stencil.py > gpurun_out/r02_stencil.log 2>&1
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_stencil_adi.py -k "cfg4_shape or 16384" > gpurun_out/adi_big.log 2>&1; echo "rc=$?" >> gpurun_out/adi_big.log
ls -la gpurun_out
