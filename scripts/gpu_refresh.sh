# Evidence refresh for the current build: full GPU parity suite, the default bench line (e2e +
# cpu baseline), per-config bench lines, the launch list (ncu gpu__time_duration) of the default
# bench command, and one full-size ncu --set full raw page per config in TRAFFIC (DRAM traffic).
set -o pipefail
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; cat gpurun_out/bench_full.json
for c in ${CFGS:-c1 c2 c4 c5}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c',d['value'],r['fused_ms_per_launch'],r['frac'],d['e2e']['value'],d['clocks'])"
done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
for c in ${TRAFFIC:-c5}; do
  P="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 900 $P > gpurun_out/plain_traffic_$c.log 2>&1 && timeout 1200 ncu --set full --clock-control none -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_full_$c $P > gpurun_out/ncu_traffic_$c.log 2>&1; echo "$c ncu rc=$?"
  ncu -i gpurun_out/prof_full_$c.ncu-rep --page raw --csv > gpurun_out/raw_full_$c.csv 2>/dev/null
  rm -f gpurun_out/prof_full_$c.ncu-rep
done
