# Round-2 evidence in one gpurun call: GPU suite, every bench line (all configs, response formats,
# SIMD formulation), the launch list of the default bench, ncu --set full of the c3 and c4 fused
# kernels, the microbenchmarks and smoke.  Outputs under gpurun_out/ (copied to profiles/ by hand).
set -o pipefail
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c3_default.json 2> gpurun_out/bench_c3_default.err; echo "bench rc=$?"; head -c 400 gpurun_out/bench_c3_default.json; echo
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c',d['value'],r['fused_ms_per_launch'],r['frac'],d['e2e']['value'],d['clocks'])"
done
for f in full compact; do
  timeout 900 python bench.py --config c3 --resp $f --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$f.json 2> gpurun_out/bench_c3_$f.err
  python -c "import json;d=json.load(open('gpurun_out/bench_c3_$f.json'));r=d['roofline'];print('c3 $f',d['value'],r['fused_ms_per_launch'],r['frac'],d['e2e']['value'])"
done
timeout 900 python bench.py --config c4 --resp full --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_full.json 2> gpurun_out/bench_c4_full.err
python -c "import json;d=json.load(open('gpurun_out/bench_c4_full.json'));r=d['roofline'];print('c4 full',d['value'],r['fused_ms_per_launch'],r['frac'],d['e2e']['value'])"
bash scripts/gpu_simd_refresh.sh
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
# full captures go to /tmp (an .ncu-rep is tens of MB; gpurun_out/ must stay under 64 MiB): the summaries,
# the per-line stall table and the traffic record are written here on the box
declare -A KN=([c3]=_ZN5wally14eval_kernel_prILi3ELi2EEEvNS_9BatchArgsE [c4]=_ZN5wally15eval_kernel_p8tILi4ELi1EEEvNS_9BatchArgsE [c5]=_ZN5wally14eval_kernel_prILi2ELi2EEEvNS_9BatchArgsE)
for c in c3 c4 c5; do
  P="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 600 $P > gpurun_out/plain_full_$c.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o /tmp/prof_final_$c $P > gpurun_out/ncu_final_$c.log 2>&1; echo "$c ncu rc=$?"
  python scripts/ncu_summary.py /tmp/prof_final_$c.ncu-rep > gpurun_out/ncu_summary_$c.txt 2>&1
  python scripts/ncu_lines.py /tmp/prof_final_$c.ncu-rep paper_2406_06761_b200/libwally.so ${KN[$c]} 30 > gpurun_out/ncu_lines_$c.txt 2>&1
  cp profiles/ncu_fused_traffic.json gpurun_out/ncu_fused_traffic.json 2>/dev/null
  python scripts/update_traffic.py $c /tmp/prof_final_$c.ncu-rep 2 > /dev/null 2>&1 && cp profiles/ncu_fused_traffic.json gpurun_out/ncu_fused_traffic.json
done
./paper_2406_06761_b200/intpipe_bench > gpurun_out/intpipe.jsonl 2>&1
./paper_2406_06761_b200/imma_bench > gpurun_out/imma.jsonl 2>&1
./paper_2406_06761_b200/tc_ntt_bench --reps 16 --mma-only > gpurun_out/tc_ntt.jsonl 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference rc=$?"; head -c 300 gpurun_out/bench_reference.json; echo
