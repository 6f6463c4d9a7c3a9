python -c "import torch; torch.zeros(1).cuda()"
for i in $(seq 1 10); do
  out=$(PB_TP_P2G=2 timeout 60 python tools/tp_repeat_many.py 512 262144 1 300 2>&1 | grep -E "done|pentab error|AcceleratorError" | head -1); echo "p2g $i: ${out:-HANG}"
done
PB_TP_P2G=2 python tools/tp_check.py 512 262144; PB_TP_P2G=2 python tools/sweep_shapes.py 8192:8192 2>&1 | tail -1
