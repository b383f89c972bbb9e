# A/B an environment knob on the headline solve: bash scripts/ab_env.sh VAR val1 val2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --no-cpu --no-kernels --no-extra --steps 10 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$var" "$v" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/ab.json"))
    print(sys.argv[1], sys.argv[2], "H_MG", round(d["ms_per_step"], 3), "D_MG", round(d["fp64_baseline"]["seconds"] * 1e3, 3),
          "ratio", round(d["fp64_baseline"]["speedup_mixed_vs_fp64"], 3))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e, open("gpurun_out/ab.err").read()[-500:])
PY
done
