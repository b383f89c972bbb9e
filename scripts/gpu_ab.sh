# A/B of an env knob on the bench line: bash scripts/gpu_ab.sh VAR v1 v2 ...
var=$1; shift
for rep in 1 2; do for v in "$@"; do
env $var=$v timeout 300 python bench.py --no-cpu --no-kernels --steps 10 > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$var=$v', round(d['ms_per_step'],3), round(d['fp64_baseline']['seconds']*1e3,3), d['iterations'])"
done; done
