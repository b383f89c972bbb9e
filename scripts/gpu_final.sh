# Round-end evidence run: GPU tests, bench (with the CPU baseline and extra
# configs), an ncu launch list of one solve and one ncu --set full capture of
# the dominant kernel; files under gpurun_out/final/
set -x
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 2>&1 | tail -30 > gpurun_out/final/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_h_mg_257.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 --no-kernels --no-graph --no-extra > gpurun_out/final/launches.log 2>&1
python scripts/launch_summary.py gpurun_out/final/launches_h_mg_257.csv > gpurun_out/final/launches_h_mg_257_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plane -c 1 -o gpurun_out/final/prof_jacobi python bench.py --only-kernels --kernel-reps 1 --steps 1 --warmup 0 > gpurun_out/final/ncu_jacobi.log 2>&1
tail -3 gpurun_out/final/pytest_gpu.txt; cut -c1-300 gpurun_out/final/bench.json; head -12 gpurun_out/final/launches_h_mg_257_summary.txt
