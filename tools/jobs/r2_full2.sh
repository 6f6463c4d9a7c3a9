mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()"
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_coarsen.py > gpurun_out/coarsen_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/coarsen_pytest.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
