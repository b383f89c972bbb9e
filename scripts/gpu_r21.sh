for v in 0 5 8 9; do
MPMG_UPD_VARIANT=$v timeout 300 python bench.py --no-cpu --no-fp64 --no-kernels --steps 5 > gpurun_out/bench_u$v.json 2> gpurun_out/bench_u$v.err
python -c "
import json; d=json.load(open('gpurun_out/bench_u$v.json')); print($v, d['ms_per_step'], d['iterations'])"
done
