timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "v_cycle or coarse or ir_solve" 2>&1 | tail -2
python scripts/coarse_probe.py 257 8 h_mg 2>&1 | tail -21
MPMG_COARSE_DEBUG=5 python scripts/coarse_probe.py 257 8 h_mg 2>&1 | head -12
timeout 300 python bench.py --no-cpu --no-kernels --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['fp64_baseline']['seconds'], d['iterations'])"
