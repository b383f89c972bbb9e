timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['fp64_baseline'], d['iterations'], {k: round(v['avg_us'],1) for k,v in d['kernels'].items()})"
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -3
