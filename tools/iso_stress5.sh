python -c "import torch; torch.zeros(1).cuda()"
for i in $(seq 1 6); do
  out=$(timeout 60 python tools/tp_repeat_many.py 512 262144 1 300 2>&1 | grep -E "done|pentab error|AcceleratorError" | head -1); echo "auto-big $i: ${out:-HANG}"
done
for i in 1 2 3; do
  out=$(PB_SOLVER=tp timeout 60 python tools/tp_repeat.py 8192 8192 3000 nosync 2>&1 | grep -E "done|pentab error|AcceleratorError" | head -1); echo "bench-shape $i: ${out:-HANG}"
done
python tools/sweep_shapes.py 8192:8192 512:262144 2>&1 | tail -2
