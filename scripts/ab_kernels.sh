# A/B an environment knob on the per-kernel timings (bench.py --only-kernels):
#   bash scripts/ab_kernels.sh VAR val1 val2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --only-kernels > gpurun_out/abk.json 2> gpurun_out/abk.err
  python - "$var" "$v" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/abk.json"))
    print(sys.argv[1], sys.argv[2], {k: round(v["avg_us"], 2) for k, v in d.items() if isinstance(v, dict) and "avg_us" in v})
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e, open("gpurun_out/abk.err").read()[-400:])
PY
done
