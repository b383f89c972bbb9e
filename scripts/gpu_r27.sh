for rep in 1 2; do for v in 0 1; do
MPMG_DEF64_SHAPE=$v timeout 300 python bench.py --no-cpu --steps 10 > gpurun_out/bench_s$v.json 2> gpurun_out/bench_s$v.err
python -c "
import json; d=json.load(open('gpurun_out/bench_s$v.json')); print($v, round(d['ms_per_step'],3), round(d['fp64_baseline']['seconds']*1e3,3), {k: round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done; done
