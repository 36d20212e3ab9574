# A/B timing of library variants: LIBS="a.so b.so" CFGS="c3 c4" [EXTRA="--resp full"] bash scripts/ab_bench.sh
mkdir -p gpurun_out
for cfg in ${CFGS:-c4}; do
for lib in ${LIBS}; do
  WALLY_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline ${EXTRA} > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));r=d['roofline'];print('$cfg','$lib',r['fused_ms_per_launch'],r['frac'],d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done; done
