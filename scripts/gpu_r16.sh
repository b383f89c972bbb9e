for w in 1 2 4 8; do
MPMG_OUTER_WAVES=$w timeout 300 python bench.py --no-cpu --no-fp64 --steps 5 > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err
python - <<PY
import json; d=json.load(open('gpurun_out/bench_w$w.json')); k=d['kernels']
print($w, round(d['ms_per_step'],3), {n: round(k[n]['avg_us'],1) for n in ('jacobi_fine','update_rc','downcast','defect64')})
PY
done
