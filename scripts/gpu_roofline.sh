# Hierarchical roofline captures (one solve each, no graph) + peaks probe +
# the dominant kernel's full ncu capture; summaries into gpurun_out/roof/
set -x
mkdir -p gpurun_out/roof
./scripts/probe_peaks.bin > gpurun_out/roof/peaks.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_bytes.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 --no-kernels --no-graph --no-extra"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/roof/h_mg_257.csv $B > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/roof/d_mg_257.csv $B --variant d_mg > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/roof/hsd_mg_257.csv $B --variant hsd_mg > /dev/null 2>&1
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/roof/h_mg_2d_8193.csv $B --dim 2 --nodes 8193 > /dev/null 2>&1
for c in h_mg_257 d_mg_257 hsd_mg_257 h_mg_2d_8193; do
  python scripts/roofline_table.py gpurun_out/roof/$c.csv gpurun_out/roof/peaks.txt "$c" gpurun_out/roof/$c.json > gpurun_out/roof/$c.md 2>&1
done
cat gpurun_out/roof/peaks.txt
