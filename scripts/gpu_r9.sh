set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_h.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 --no-kernels --no-graph > gpurun_out/launches_h.log 2>&1
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json | cut -c1-300; cat gpurun_out/coarse_probe.txt
