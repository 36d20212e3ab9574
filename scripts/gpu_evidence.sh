# Evidence run for the current build: bench per config, launch list (ncu timing) of the default bench
# command, ncu --set full of the fused kernel on a c3 subset.
set -o pipefail
mkdir -p gpurun_out
for c in ${CFGS:-c3 c4 c5 c2}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c',d['value'],r['fused_ms_per_launch'],r['frac'],d['stages_ms_per_step'],d['clocks'])"
done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
P="python bench.py --config c3 --queries 2048 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $P > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_eval_c3 $P > gpurun_out/ncu_prof.log 2>&1; echo "ncu full rc=$?"
