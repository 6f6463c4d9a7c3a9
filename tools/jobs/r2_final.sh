mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
python -c "import torch; torch.zeros(1).cuda()"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_launches.csv python bench.py --steps 5 --warmup 3 --adi-steps 5 --no-cpu > gpurun_out/r02d_ncu_launch.log 2>&1
full() {  # name, kernel regex, skip, count, command...
  n=$1; k=$2; s=$3; c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/$n -f "$@" > gpurun_out/$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/$n.raw.csv 2>/dev/null
}
full r02d_solve tp_ 6 3 python tools/prof_solve.py 8192 f64 4
full r02d_solve32 tp_ 6 3 python tools/prof_solve.py 8192 f32 4
full r02d_adi . 18 6 python tools/prof_adi_step.py
full r02d_ch1d fh_ 2 1 python tools/prof_ch1d.py
full r02d_stencil stencil 0 1 python tools/prof_stencil.py
du -sh gpurun_out
