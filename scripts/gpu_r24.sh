MPMG_DIRECT_MAX_P=256 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "level_kernels or v_cycle or ir_solve" 2>&1 | tail -3
for m in 0 64 128 256; do
MPMG_DIRECT_MAX_P=$m timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_d$m.json 2> gpurun_out/bench_d$m.err
MPMG_DIRECT_MAX_P=$m python scripts/level_probe.py 20 > gpurun_out/level_d$m.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_d$m.json')); print($m, d['ms_per_step'], d['fp64_baseline']['seconds'], d['iterations'])"
grep -E "^ +(257|129|65|33) +(jacobi|jacobi0|defect) " gpurun_out/level_d$m.txt | tr '\n' ' '; echo
done
