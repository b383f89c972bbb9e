set -x
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "v_cycle or coarse or ir_solve or deferred" 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
MPMG_COARSE_CLUSTER=8 timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_c8.json 2> gpurun_out/bench_c8.err
MPMG_COARSE_CLUSTER=0 timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err
cat gpurun_out/pytest_gpu.txt; for f in bench bench_c8 bench_c0; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['ms_per_step'], d['fp64_baseline']['seconds'], d['iterations'])"; done; cat gpurun_out/coarse_probe.txt; tail -3 gpurun_out/bench.err
