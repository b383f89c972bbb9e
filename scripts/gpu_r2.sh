set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_ftz scripts/probe_ftz.cu && /tmp/probe_ftz > gpurun_out/probe_ftz.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_h.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 --no-kernels --no-graph > gpurun_out/launches_h.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_d.csv python bench.py --steps 1 --warmup 0 --no-cpu --variant d_mg --no-kernels --no-graph > gpurun_out/launches_d.log 2>&1
cat gpurun_out/probe_ftz.txt
