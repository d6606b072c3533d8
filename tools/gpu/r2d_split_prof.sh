mkdir -p gpurun_out/r2d
export TSV_NO_BUILD=1
for mode in 1 0; do
TSV_AS_SPLIT=$mode timeout 900 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_registers --clock-control none -k 'regex:^(as_|gemm_nt|tc_local|oz_|cg_)' --launch-skip 300 -c 120 --csv --log-file gpurun_out/r2d/launches_split$mode.csv python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2d/ncu$mode.log 2>&1
echo "ncu$mode rc=$?"
done
for v in "TSV_AS_SPLIT=1 TSV_NO_PDL=1" "TSV_AS_SPLIT=1 TSV_AS_S=2" "TSV_AS_SPLIT=0 TSV_AS_S=2"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2d/b.json 2>/dev/null
  echo "$v rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2d/b.json').read().strip().splitlines()[-1]);print(d['value'],d['config']['iterations'],d['phase_ms'],d['precond'])"
done
