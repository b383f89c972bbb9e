for p in 0 1 2; do
MPMG_COARSE_PER_SM=$p python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe_p$p.txt 2>&1
MPMG_COARSE_PER_SM=$p timeout 300 python bench.py --no-cpu --no-kernels --steps 5 > gpurun_out/bench_p$p.json 2> gpurun_out/bench_p$p.err
python -c "
import json; d=json.load(open('gpurun_out/bench_p$p.json')); print($p, d['ms_per_step'], d['fp64_baseline']['seconds'])"
tail -2 gpurun_out/coarse_probe_p$p.txt
done
