# many back-to-back default-path solves per process, one process per variant
# (PB_TP_VAR bits); reports done / error / hang (empty)
python -c "import torch; torch.zeros(1).cuda()"   # warm the image
for d in "$@"; do
  out=$(PB_TP_VAR=$d timeout 40 python tools/tp_repeat.py 8192 8192 3000 nosync 2>&1 | grep -v Warn | grep -E "done|Error|error" | head -1)
  echo "var $d : ${out:-HANG}"
done
