# Quick iteration on one B200: GPU parity (fast subset unless FULL=1), bench per library
# variant (no e2e / cpu baseline), int-pipe microbench, optional ncu --set full of the fused kernel.
set -o pipefail
mkdir -p gpurun_out
./paper_2406_06761_b200/intpipe_bench > gpurun_out/intpipe.jsonl 2>&1; cat gpurun_out/intpipe.jsonl
if [ "${FULL:-0}" = "1" ]; then K=""; else K="-k not full_config"; fi
timeout 1200 python -m pytest tests -m gpu -x -q "$K" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
for lib in ${LIBS:-paper_2406_06761_b200/libwally.so}; do
  for cfg in ${CFGS:-c3}; do
  echo "== $lib $cfg"
  WALLY_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; tail -2 gpurun_out/bench_iter.err
  python -c "import json;d=json.load(open('gpurun_out/bench_iter.json'));r=d['roofline'];print('value',d['value'],'fused_ms',r['fused_ms_per_launch'],'frac',r['frac'],'stages',d['stages_ms_per_step'],'clk',d['clocks'])"
  done
done
P="python bench.py --config ${PCFG:-c3} --queries 2048 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
if [ "${PROFILE:-1}" = "1" ]; then
timeout 600 $P > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_iter $P > gpurun_out/ncu_prof.log 2>&1; echo "ncu rc=$?"
fi
