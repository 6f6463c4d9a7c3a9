mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 400 ncu --set full --import-source on --clock-control none -k regex:tp_p2 -s 1 -c 1 -o gpurun_out/tp8192 -f python tools/prof_solve.py 8192 f64 3 > gpurun_out/tp8192_ncu.txt 2>&1
