# Everything the profiles/ directory holds, in one gpurun call (about 20 GPU-minutes):
# GPU suite, the default bench line, per-config lines, SIMD lines, the launch list,
# DRAM traffic of c3/c4/c5, ncu --set full of the c3 and c4 fused kernels, the microbenchmarks.
set -o pipefail
mkdir -p gpurun_out
CFGS="c1 c2 c4 c5" TRAFFIC="c3 c4 c5" bash scripts/gpu_refresh.sh
bash scripts/gpu_simd_refresh.sh
for c in c3 c4; do
  P="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_final_$c $P > gpurun_out/ncu_final_$c.log 2>&1; echo "$c ncu rc=$?"
done
./paper_2406_06761_b200/intpipe_bench > gpurun_out/intpipe.jsonl 2>&1
./paper_2406_06761_b200/imma_bench > gpurun_out/imma.jsonl 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
