set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "deferred or ir_solve" 2>&1 | tail -15 > gpurun_out/pytest_defer.txt
timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
MPMG_DEFER_U=0 timeout 300 python bench.py --no-cpu --no-kernels --no-fp64 --steps 5 > gpurun_out/bench_nodefer.json 2> gpurun_out/bench_nodefer.err
tail -5 gpurun_out/pytest_defer.txt; cut -c1-400 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_nodefer.json; tail -3 gpurun_out/bench.err
