# SIMD-formulation bench lines for every config, with e2e and the oracle baseline.
set -o pipefail
mkdir -p gpurun_out
for c in ${CFGS:-c1 c2 c3 c4 c5}; do
  timeout 900 python bench.py --path simd --config $c --steps 3 --warmup 3 > gpurun_out/simd_$c.json 2> gpurun_out/simd_$c.err
  echo "$c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/simd_$c.json'));print('$c',d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d.get('cpu_baseline',{}).get('value'),d['clocks'])"
done
