set -x
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe.txt 2>&1
MPMG_COARSE_CLUSTER=0 python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe_coop.txt 2>&1
timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
MPMG_COARSE_CLUSTER=0 timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_coop.json 2> gpurun_out/bench_coop.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt; cut -c1-300 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_coop.json; cat gpurun_out/coarse_probe.txt gpurun_out/coarse_probe_coop.txt
