mkdir -p gpurun_out/r2k
export TSV_NO_BUILD=1
timeout 600 python -m pytest tests/test_schwarz.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_online_dt.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2k/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -1 gpurun_out/r2k/pytest_quick.log
b() { env $1 timeout 600 python bench.py --config $2 --steps $3 --warmup 5 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2k/b.json 2>gpurun_out/r2k/b.err; echo "cfg$2 $1 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2k/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'],d['clocks']['samples'])" || tail -3 gpurun_out/r2k/b.err; }
for c in 0 1 2; do b "TSV_K1_SPLITK=1" $c 200; b "TSV_K1_SPLITK=0" $c 200; done
b "TSV_AS_SYMV_ONE=0" 3 5; b "TSV_AS_SYMV_ONE=1" 3 5; b "TSV_AS_SYMV_CTAS=4" 3 5; b "TSV_AS_SYMV_CTAS=16" 3 5
