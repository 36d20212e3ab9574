# quick iteration: GPU parity (fast subset), bench (no e2e/cpu) per library variant, ncu full on the fused kernel
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_config" 2>&1 | tail -3
for lib in ${LIBS:-paper_2406_06761_b200/libwally.so}; do
  echo "== $lib"
  WALLY_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; tail -2 gpurun_out/bench_iter.err
  python -c "import json;d=json.load(open('gpurun_out/bench_iter.json'));r=d['roofline'];print('value',d['value'],'fused_ms',r['fused_ms_per_launch'],'frac',r['frac'],'stages',d['stages_ms_per_step'],'clk',d['clocks'])"
done
P="python bench.py --config c3 --queries 2048 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
if [ "${PROFILE:-1}" = "1" ]; then
$P > gpurun_out/plain_prof.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_iter $P > gpurun_out/ncu_prof.log 2>&1; echo "ncu rc=$?"
fi
