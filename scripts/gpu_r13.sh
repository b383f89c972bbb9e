set -x
python scripts/level_probe.py 20 > gpurun_out/level_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/level_probe.txt
