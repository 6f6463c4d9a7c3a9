# batched (count > 1) two-pass solves and cfg4 ADI runs, repeated (dev stress test)
python -c "import torch; torch.zeros(1).cuda()"
for i in $(seq 1 ${1:-6}); do
  out=$(timeout 60 python tools/tp_repeat_many.py 512 512 512 400 2>&1 | grep -E "done|rror" | head -1); echo "tpmany $i: ${out:-HANG}"
done
for i in $(seq 1 ${2:-6}); do
  out=$(timeout 60 python tools/adi_sweep.py 2>&1 | grep -E "ms/step|rror" | head -1); echo "adi $i: ${out:-HANG}"
done
