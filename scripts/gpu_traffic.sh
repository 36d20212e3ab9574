# DRAM traffic of one full-size fused-kernel launch per config (ncu --set full), for bench.py's roofline.traffic
set -o pipefail
mkdir -p gpurun_out
for c in ${CFGS:-c3}; do
  P="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 900 $P > gpurun_out/plain_traffic_$c.log 2>&1 && timeout 1200 ncu --set full --clock-control none -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_full_$c $P > gpurun_out/ncu_traffic_$c.log 2>&1; echo "$c ncu rc=$?"
done
