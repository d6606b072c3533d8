mkdir -p gpurun_out/r2o
export TSV_NO_BUILD=1
timeout 1200 python -m pytest tests/test_schwarz.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_online_dt.py tests/test_variants.py tests/test_integration.py "tests/test_gpu_configs.py::test_config1_reference_parity" -m gpu -x -q -p no:cacheprovider > gpurun_out/r2o/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -3 gpurun_out/r2o/pytest_quick.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
b() { env $1 timeout 600 python bench.py --config $2 --steps $3 --warmup 5 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2o/b.json 2>gpurun_out/r2o/b.err; echo "cfg$2 $1 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2o/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'],d['clocks']['samples'],d['gpu_launches'])" || tail -5 gpurun_out/r2o/b.err; }
for c in 0 1; do b "TSV_SMALL_PCG=1" $c 300; b "TSV_SMALL_PCG=0" $c 300; done
b "TSV_SMALL_PCG=1" 2 50; b "TSV_SMALL_PCG=0" 2 50
