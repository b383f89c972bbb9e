set -x
timeout 900 python -m pytest tests/test_dist.py -m gpu -q --timeout 600 2>&1 | tail -40 > gpurun_out/pytest_dist.txt
for cp in 32768 262144 2100000; do
  MPMG_COARSE_POINTS=$cp timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_cp$cp.json 2> gpurun_out/bench_cp$cp.err
done
MPMG_COARSE_POINTS=32768 MPMG_COARSE_DEBUG=1 timeout 300 python bench.py --no-cpu --no-kernels --no-fp64 --steps 1 --warmup 0 > gpurun_out/coarse_debug.txt 2>&1
MPMG_COARSE_POINTS=2100000 MPMG_COARSE_DEBUG=1 timeout 300 python bench.py --no-cpu --no-kernels --no-fp64 --steps 1 --warmup 0 > gpurun_out/coarse_debug2.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 --deselect tests/test_dist.py 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_dist.txt | tail -5; grep -h value gpurun_out/bench_cp*.json | cut -c1-300
