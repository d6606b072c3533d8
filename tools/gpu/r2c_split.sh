# split Schwarz loop: correctness + A/B timing at config 3
mkdir -p gpurun_out/r2c
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_schwarz.py tests/test_gpu_parity.py tests/test_online_dt.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -3 gpurun_out/r2c/pytest_quick.log
for mode in 0 1; do
  TSV_AS_SPLIT=$mode timeout 600 python bench.py --steps 3 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c/bench_split$mode.json 2> gpurun_out/r2c/bench_split$mode.err
  echo "bench split=$mode rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2c/bench_split$mode.json').read().strip().splitlines()[-1]);print(d['value'],d['config']['iterations'],d['phase_ms'])"
done
TSV_AS_SPLIT=1 TSV_NO_FUSED_GU=1 timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c/bench_cfg2.json 2>&1
echo "bench cfg2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c/launches.csv python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c/ncu.log 2>&1
echo "ncu rc=$?"
