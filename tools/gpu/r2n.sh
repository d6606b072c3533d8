mkdir -p gpurun_out/r2n
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_schwarz.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_online_dt.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2n/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -1 gpurun_out/r2n/pytest_quick.log
b() { env $1 timeout 600 python bench.py --config $2 --steps $3 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2n/b.json 2>gpurun_out/r2n/b.err; echo "cfg$2 $1 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2n/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'])" || tail -3 gpurun_out/r2n/b.err; }
for c in 3 4 1; do b "TSV_AS_SCATTER_NODE=0" $c 5; b "TSV_AS_SCATTER_NODE=1" $c 5; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(as_|gemm_nt|tc_local|oz_|cg_)' --launch-skip 300 -c 120 --csv --log-file gpurun_out/r2n/launches.csv python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2n/ncu.log 2>&1
echo "ncu rc=$?"
