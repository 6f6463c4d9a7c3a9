mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_ch1d.py -k "large_and_long" > gpurun_out/ch1d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ch1d_pytest.log
