set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_h.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 --no-kernels --no-graph > gpurun_out/launches_h.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_h.csv > gpurun_out/launches_h_summary.txt 2>&1
head -60 gpurun_out/launches_h_summary.txt
