set -x
for v in 0 6 7; do MPMG_PLANE_VARIANT=$v timeout 300 python bench.py --only-kernels --steps 5 > gpurun_out/kern_v$v.json 2>gpurun_out/kern_v$v.err; done
timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python scripts/coarse_probe.py 257 8 h_mg > gpurun_out/coarse_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt; for v in 0 6 7; do python -c "import json;d=json.load(open('gpurun_out/kern_v$v.json'));print($v, {k:round(x['avg_us'],2) for k,x in d['kernels'].items() if isinstance(x,dict)})"; done; cut -c1-300 gpurun_out/bench.json; cat gpurun_out/coarse_probe.txt
