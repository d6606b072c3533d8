mkdir -p gpurun_out/r2m
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_schwarz.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_variants.py tests/test_online_dt.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2m/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -1 gpurun_out/r2m/pytest_quick.log
b() { env $1 timeout 600 python bench.py --config $2 --steps $3 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2m/b.json 2>gpurun_out/r2m/b.err; echo "cfg$2 $1 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2m/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'],d['roofline']['frac'])" || tail -3 gpurun_out/r2m/b.err; }
for c in 3 4; do b "TSV_K1_TAILSPLIT=1" $c 5; b "TSV_K1_TAILSPLIT=0" $c 5; done
