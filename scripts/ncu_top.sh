# ncu --set full of one kernel matched by regex $1 (first launch of bench --only-kernels)
# usage: bash scripts/ncu_top.sh <regex> <outname>
timeout 800 ncu --set full --clock-control none --import-source on -k regex:$1 -c 1 -o gpurun_out/$2 python bench.py --only-kernels --kernel-reps 1 --steps 1 --warmup 0 > gpurun_out/$2.log 2>&1
tail -1 gpurun_out/$2.log
