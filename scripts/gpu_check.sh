set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-fp64 --no-kernels > gpurun_out/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k_downcast" -c 8 -o gpurun_out/prof_fine python bench.py --only-kernels --kernel-reps 1 > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
