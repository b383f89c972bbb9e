for v in 0 10; do
MPMG_UPD_VARIANT=$v timeout 300 python bench.py --no-cpu --no-fp64 --steps 5 > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.err
python -c "
import json; d=json.load(open('gpurun_out/bench_v$v.json')); print($v, d['ms_per_step'], d['iterations'], d['kernels']['update_r']['avg_us'])"
done
MPMG_UPD_VARIANT=10 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x --timeout 600 -k "deferred or update_r" 2>&1 | tail -2
