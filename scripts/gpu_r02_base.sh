# Round-2 baseline on a fresh box: full GPU suite, default bench line, c4 line,
# and one ncu --set full of the c4 fused kernel (L2 hit/miss breakdown).
set -o pipefail
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_base_c3.json 2> gpurun_out/r02_base_c3.err; echo "bench c3 rc=$?"; cat gpurun_out/r02_base_c3.json | head -c 600; echo
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_base_c4.json 2> gpurun_out/r02_base_c4.err; echo "bench c4 rc=$?"
P="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/r02_prof_c4 $P > gpurun_out/r02_ncu_c4.log 2>&1; echo "c4 ncu rc=$?"
