for m in 0 128 256; do
MPMG_PLANE_MIN_P=$m timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_m$m.json 2> gpurun_out/bench_m$m.err
MPMG_PLANE_MIN_P=$m python scripts/level_probe.py 20 > gpurun_out/level_m$m.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_m$m.json')); print($m, d['ms_per_step'], d['fp64_baseline']['seconds'], d['iterations'])"
grep -E "^ +(129|65|33) +(jacobi|defect) " gpurun_out/level_m$m.txt | tr '\n' ' '; echo
done
