set -x
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe.txt 2>&1
MPMG_CTA_POINTS=343 python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe_343.txt 2>&1
timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
MPMG_CTA_POINTS=343 timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_343.json 2> gpurun_out/bench_343.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "v_cycle or coarse or ir_solve" 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt; cut -c1-250 gpurun_out/bench.json; cut -c1-250 gpurun_out/bench_343.json; cat gpurun_out/coarse_probe.txt gpurun_out/coarse_probe_343.txt
