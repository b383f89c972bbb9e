set -x
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe.txt 2>&1
timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python scripts/level_probe.py 20 > gpurun_out/level_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt; cut -c1-300 gpurun_out/bench.json; cat gpurun_out/coarse_probe.txt gpurun_out/level_probe.txt
