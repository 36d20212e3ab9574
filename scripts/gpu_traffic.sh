# DRAM traffic + pipe metrics of one full-size fused-kernel launch per config (ncu --set full),
# for bench.py's roofline.traffic.  The raw page is exported on the box (small CSV) and only the
# c3 report is kept (gpurun brings back at most 64 MiB).
set -o pipefail
mkdir -p gpurun_out
for c in ${CFGS:-c3}; do
  P="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 900 $P > gpurun_out/plain_traffic_$c.log 2>&1 && timeout 1200 ncu --set full --clock-control none -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_full_$c $P > gpurun_out/ncu_traffic_$c.log 2>&1; echo "$c ncu rc=$?"
  ncu -i gpurun_out/prof_full_$c.ncu-rep --page raw --csv > gpurun_out/raw_full_$c.csv 2>/dev/null
  [ "$c" = "${KEEP:-c3}" ] || rm -f gpurun_out/prof_full_$c.ncu-rep
done
