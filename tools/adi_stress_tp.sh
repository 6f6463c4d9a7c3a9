python -c "import torch; torch.zeros(1).cuda()"
for i in $(seq 1 ${1:-12}); do
  out=$(PB_ADI_YSWEEP=tp timeout 60 python tools/adi_sweep.py 2>&1 | grep -E "ms/step|rror" | head -1)
  echo "adi-tp $i: ${out:-HANG/KILLED}"
done
