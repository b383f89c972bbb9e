# iteration check while tuning: 257^3 parity tests, then the bench line
# (device H_MG vs D_MG solve, per-kernel timings)
timeout 900 python -m pytest tests/test_gpu_parity_257.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/b.json 2> gpurun_out/b.err
python - <<'PY'
import json
d = json.load(open('gpurun_out/b.json'))
print('H_MG ms', round(d['ms_per_step'], 3), 'D_MG ms', round(d['fp64_baseline']['seconds'] * 1e3, 3), 'its',
      d['iterations'], 'ratio', round(d['fp64_baseline']['speedup_mixed_vs_fp64'], 3), 'e2e ms',
      round(d['e2e']['value'] * 1e3, 3))
for k, v in d.get('kernels', {}).items():
    print(' ', k, round(v['avg_us'], 2), 'us', round(v['achieved_gbs']), 'GB/s')
PY
