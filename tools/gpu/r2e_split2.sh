mkdir -p gpurun_out/r2e
export TSV_NO_BUILD=1
timeout 600 python -m pytest tests/test_schwarz.py tests/test_online_dt.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2e/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -2 gpurun_out/r2e/pytest_quick.log
for v in "TSV_AS_SPLIT=1" "TSV_AS_SPLIT=1 TSV_AS_S=2" "TSV_AS_SPLIT=0 TSV_AS_S=2" "TSV_AS_SPLIT=0"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2e/b.json 2>/dev/null
  echo "$v rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2e/b.json').read().strip().splitlines()[-1]);print(d['value'],d['config']['iterations'],d['phase_ms'])"
done
TSV_AS_SPLIT=1 TSV_AS_S=2 timeout 900 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_registers --clock-control none -k 'regex:^(as_|gemm_nt|tc_local|oz_|cg_)' --launch-skip 300 -c 120 --csv --log-file gpurun_out/r2e/launches_split_s2.csv python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2e/ncu.log 2>&1
echo "ncu rc=$?"
