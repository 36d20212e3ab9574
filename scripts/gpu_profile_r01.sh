set -o pipefail
./paper_2406_06761_b200/intpipe_bench > gpurun_out/intpipe.jsonl 2>&1; cat gpurun_out/intpipe.jsonl
timeout 1200 python -m pytest tests -m gpu -x -q -k "full_config" 2>&1 | tail -8
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
P="python bench.py --config c3 --queries 2048 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_prof.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_eval_c3 $P > gpurun_out/ncu_prof.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_prof.log
