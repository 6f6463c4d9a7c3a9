#!/bin/bash
# Ring-protocol stress (GPU box): long queued chains of solves in the regimes
# that faulted in round 1, each under its own timeout, plus compute-sanitizer
# synccheck / racecheck on a small shape.  Usage: bash tools/ring_stress.sh RUNS
R=${1:-5}
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
for i in $(seq 1 $R); do
  out=$(timeout 120 python tools/tp_repeat_many.py 512 262144 1 2000 2>&1 | grep -E "done|rror" | head -1); echo "512x262144 count1 x2000 run $i: ${out:-HANG}"
done
for i in $(seq 1 $R); do
  out=$(timeout 120 python tools/tp_repeat_many.py 512 512 512 2000 2>&1 | grep -E "done|rror" | head -1); echo "512x512 count512 x2000 run $i: ${out:-HANG}"
done
for i in $(seq 1 $R); do
  out=$(timeout 120 python tools/tp_repeat_many.py 512 512 3 2000 2>&1 | grep -E "done|rror" | head -1); echo "512x512 count3 x2000 run $i: ${out:-HANG}"
done
for i in $(seq 1 $R); do
  out=$(timeout 120 python tools/adi_sweep.py 2>&1 | grep -E "ms/step|rror" | head -1); echo "adi cfg4 x23 run $i: ${out:-HANG}"
done
for tool in synccheck racecheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/tp_repeat.py 300 96 3 > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitizer_$tool.txt | tail -1)"
done
