# One ncu --set full capture of the fused kernel of one config (after a plain run of the same command).
# Usage: CFG=c4 TAG=v5 [LIB=variants/lib_x.so] bash scripts/gpu_ncu1.sh
set -o pipefail
mkdir -p gpurun_out
export WALLY_LIB=$PWD/${LIB:-paper_2406_06761_b200/libwally.so}
P="python bench.py --config ${CFG:-c4} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $P > gpurun_out/ncu_plain_${TAG}.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} $P > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
