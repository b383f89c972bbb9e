set -x
timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
MPMG_PDL=0 timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_nopdl.json 2> gpurun_out/bench_nopdl.err
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt; cut -c1-600 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_nopdl.json; cat gpurun_out/coarse_probe.txt
