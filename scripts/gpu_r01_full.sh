# Round-1 GPU evidence run: int-pipe microbench, full GPU parity suite, bench line,
# launch list (ncu, gpu__time_duration) of the bench command, ncu --set full of the fused kernel.
set -o pipefail
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 ./paper_2406_06761_b200/intpipe_bench > gpurun_out/intpipe.jsonl 2>&1; cat gpurun_out/intpipe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; cat gpurun_out/bench_full.json
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
P="python bench.py --config c3 --queries 2048 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $P > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_eval_c3 $P > gpurun_out/ncu_prof.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_prof.log
