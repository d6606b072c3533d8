mkdir -p gpurun_out/r2j
export TSV_NO_BUILD=1
timeout 600 python -m pytest tests/test_schwarz.py tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2j/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -1 gpurun_out/r2j/pytest_quick.log
for c in 0 1 2; do for v in "TSV_K1_SPLITK=1" "TSV_K1_SPLITK=0"; do
  env $v timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2j/b.json 2>/dev/null
  echo "cfg$c $v rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2j/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'],d['clocks'])"
done; done
