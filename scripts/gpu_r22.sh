for z in 1 2 4; do
MPMG_ZMIN_SMALL=$z timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_z$z.json 2> gpurun_out/bench_z$z.err
MPMG_ZMIN_SMALL=$z python scripts/level_probe.py 20 > gpurun_out/level_z$z.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_z$z.json')); print($z, d['ms_per_step'], d['fp64_baseline']['seconds'], d['iterations'])"
grep -E "^ +(129|65|33) " gpurun_out/level_z$z.txt | tr '\n' ' '; echo
done
