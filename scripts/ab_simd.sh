# A/B timing of library variants on the SIMD formulation: LIBS="a.so b.so" CFGS="c3" bash scripts/ab_simd.sh
mkdir -p gpurun_out
for cfg in ${CFGS:-c3}; do
for lib in ${LIBS}; do
  WALLY_LIB=$PWD/$lib timeout 900 python bench.py --path simd --config $cfg --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abs.json 2>gpurun_out/abs.err
  python -c "import json;d=json.load(open('gpurun_out/abs.json'));print('simd','$cfg','$lib',d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['clocks']['reasons'])" || tail -3 gpurun_out/abs.err
done; done
