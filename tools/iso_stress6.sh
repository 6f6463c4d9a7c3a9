python -c "import torch; torch.zeros(1).cuda()"
for i in $(seq 1 6); do
  out=$(PB_TP_GMAJ=1 timeout 60 python tools/tp_repeat_many.py 512 262144 1 600 2>&1 | grep -E "done|pentab error|AcceleratorError" | head -1); echo "gmaj $i: ${out:-HANG}"
done
PB_TP_GMAJ=1 python tools/tp_check.py 512 262144; PB_TP_GMAJ=1 python tools/tp_check.py 1000 300; PB_TP_GMAJ=1 python tools/sweep_shapes.py 512:262144 8192:8192 2>&1 | tail -2
