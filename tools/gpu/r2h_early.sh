mkdir -p gpurun_out/r2h
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_schwarz.py tests/test_online_dt.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_variants.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2h/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -2 gpurun_out/r2h/pytest_quick.log
for c in 3 4; do for v in "TSV_AS_EARLY_COARSE=1" "TSV_AS_EARLY_COARSE=0"; do
  env $v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2h/b.json 2>/dev/null
  echo "cfg$c $v rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2h/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'])"
done; done
