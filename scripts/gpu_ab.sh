# A/B timing of library variants: for each "lib:config" pair, one bench line (no e2e / cpu baseline).
# Usage: PAIRS="paper_2406_06761_b200/libwally.so:c4 variants/lib_x.so:c4" bash scripts/gpu_ab.sh
set -o pipefail
mkdir -p gpurun_out
for pair in $PAIRS; do
  lib=${pair%%:*}; cfg=${pair##*:}
  tag=$(basename $lib .so)_$cfg
  WALLY_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));r=d['roofline'];print('$tag',d['value'],'fused_ms',r['fused_ms_per_launch'],'frac',r['frac'],'clk',d['clocks']['sm_mhz'],d['clocks']['reasons'])" || tail -3 gpurun_out/ab_$tag.err
done
