# Refresh of the evidence that depends on the v4 fused kernel after the DESIGN.md section 14 fix: GPU suite,
# default bench line, c3 full responses, launch list of the default bench, L = 2 state in TMEM vs registers (A/B).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c3_default.json 2> gpurun_out/bench_c3_default.err; echo "bench rc=$?"; head -c 300 gpurun_out/bench_c3_default.json; echo
timeout 900 python bench.py --config c3 --resp full --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_full.json 2> gpurun_out/bench_c3_full.err
python -c "import json;d=json.load(open('gpurun_out/bench_c3_full.json'));r=d['roofline'];print('c3 full',d['value'],r['fused_ms_per_launch'],r['frac'],d['e2e']['value'])"
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python scripts/launch_summary.py gpurun_out/launches_c3.csv > gpurun_out/launches_c3.txt 2>&1; tail -8 gpurun_out/launches_c3.txt
LIBS="paper_2406_06761_b200/libwally.so variants/libwally_tml2.so paper_2406_06761_b200/libwally.so variants/libwally_tml2.so" CFGS="c5" EXTRA="--resp full" STEPS=6 bash scripts/ab_bench.sh
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
