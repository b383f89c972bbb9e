# Round-end evidence run: GPU tests, bench (with the CPU baseline), the
# reference arm, an ncu launch list of one solve, one ncu --set full capture of
# the finest-level plane kernels, the coarse-kernel and per-level probes.
set -x
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -30 > gpurun_out/final/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_h_mg_257.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 --no-kernels --no-graph > gpurun_out/final/launches.log 2>&1
python scripts/launch_summary.py gpurun_out/final/launches_h_mg_257.csv > gpurun_out/final/launches_h_mg_257_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_plane -c 8 -o gpurun_out/final/prof_plane python bench.py --only-kernels --kernel-reps 1 --steps 1 --warmup 0 > gpurun_out/final/ncu_plane.log 2>&1
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/final/coarse_probe_h_mg.txt 2>&1
python scripts/coarse_probe.py 257 8 d_mg > gpurun_out/final/coarse_probe_d_mg.txt 2>&1
python scripts/level_probe.py 20 > gpurun_out/final/level_probe.txt 2>&1
tail -3 gpurun_out/final/pytest_gpu.txt; cut -c1-400 gpurun_out/final/bench.json; cut -c1-300 gpurun_out/final/bench_reference.json; head -30 gpurun_out/final/launches_h_mg_257_summary.txt
