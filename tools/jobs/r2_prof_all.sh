mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$t.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$t.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 5 --warmup 3 --adi-steps 5 --no-cpu > gpurun_out/r02_ncu_launch.log 2>&1
full() {  # name, kernel regex, skip, count, command...
  n=$1; k=$2; s=$3; c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/$n -f "$@" > gpurun_out/$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/$n.raw.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page details --csv > gpurun_out/$n.details.csv 2>/dev/null
}
full r02_solve tp_ 6 3 python tools/prof_solve.py 8192 f64 4
full r02_solve32 tp_ 6 3 python tools/prof_solve.py 8192 f32 4
full r02_adi . 12 4 python tools/prof_adi_step.py
full r02_ch1d fh_ 2 1 python tools/prof_ch1d.py
full r02_stencil stencil 0 1 python tools/prof_stencil.py
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_stencil_adi.py -k "cfg4_shape or 16384" > gpurun_out/adi_big.log 2>&1; echo "rc=$?" >> gpurun_out/adi_big.log
du -sh gpurun_out; ls -la gpurun_out
