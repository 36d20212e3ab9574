# Soak of the random-shape parity test (tests/test_gpu_fuzz.py) on the GPU box:
#   CASES=240 SEED=1 [BIG=1: every case a large batch] bash scripts/gpu_fuzz.sh   -> gpurun_out/fuzz.log
mkdir -p gpurun_out
WALLY_FUZZ_BIG=${BIG:-0} WALLY_FUZZ_CASES=${CASES:-240} WALLY_FUZZ_SIMD_CASES=${SIMD_CASES:-40} WALLY_FUZZ_SEED=${SEED:-1} timeout ${LIMIT:-2400} \
  python -m pytest tests/test_gpu_fuzz.py -m gpu -q -s 2>&1 | grep -v "^$" > gpurun_out/fuzz.log
echo "fuzz rc=${PIPESTATUS[0]}" >> gpurun_out/fuzz.log
tail -5 gpurun_out/fuzz.log
