# repeated cfg4 ADI runs (dev stress test): bash tools/adi_stress.sh RUNS
python -c "import torch; torch.zeros(1).cuda()"
for i in $(seq 1 ${1:-8}); do
  out=$(timeout 60 python tools/adi_sweep.py 2>&1 | grep -E "ms/step|rror" | head -1)
  echo "run $i: ${out:-HANG/KILLED}"
done
