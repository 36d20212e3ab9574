# int-pipe / TMEM microbenchmarks + ncu of three of them (short run)
set -o pipefail
mkdir -p gpurun_out
./paper_2406_06761_b200/intpipe_bench > gpurun_out/intpipe.jsonl 2>&1; cat gpurun_out/intpipe.jsonl
M="./paper_2406_06761_b200/intpipe_bench 4096"
timeout 120 $M > gpurun_out/micro_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:bench_kernel -c 16 -o gpurun_out/prof_micro $M > gpurun_out/ncu_micro.log 2>&1; echo "ncu rc=$?"
