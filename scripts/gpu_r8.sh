set -x
for v in 0 1 2 3 4 5; do
  MPMG_PLANE_VARIANT=$v timeout 300 python bench.py --only-kernels --kernel-reps 30 > gpurun_out/kern_v$v.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_restrict|k_prolong8|k_downcast8|k_jacobi_zero8" -c 8 -o gpurun_out/prof_xfer python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 --no-kernels --no-graph > gpurun_out/ncu_xfer.log 2>&1
timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for v in 0 1 2 3 4 5; do python -c "import json;d=json.load(open('gpurun_out/kern_v$v.json'));print($v, round(d['jacobi_fine']['avg_us'],2))"; done
cat gpurun_out/bench.json | cut -c1-400
