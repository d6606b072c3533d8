mkdir -p gpurun_out/r2i
export TSV_NO_BUILD=1
timeout 600 python -m pytest tests/test_schwarz.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2i/pytest_quick.log 2>&1
echo "pytest_quick_rc=$?"; tail -1 gpurun_out/r2i/pytest_quick.log
for v in "TSV_AS_RESTRICT_CTA=0" "TSV_AS_RESTRICT_CTA=1"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2i/b.json 2>/dev/null
  echo "$v rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2i/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'])"
done
TSV_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2i/timing.json 2> gpurun_out/r2i/timing.err
grep -E "schwarz2|build_schwarz2|set_layout|set_bc" gpurun_out/r2i/timing.err | tail -40
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(as_|gemm_nt|tc_local|oz_|cg_)' --launch-skip 300 -c 120 --csv --log-file gpurun_out/r2i/launches.csv python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2i/ncu.log 2>&1
echo "ncu rc=$?"
