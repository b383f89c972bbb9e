# quick GPU check used while tuning: the solve-level parity tests and a bench line
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "ir_solve or deferred or final_residual or v_cycle" 2>&1 | tail -3
timeout 300 python bench.py --no-cpu --no-kernels --steps 10 > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(round(d['ms_per_step'],3), round(d['fp64_baseline']['seconds']*1e3,3), d['iterations'], d['fp64_baseline']['speedup_mixed_vs_fp64'])"
