mkdir -p gpurun_out
P="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $P > gpurun_out/plain_c4.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_c4_v6 $P > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
