mkdir -p gpurun_out/r2f
export TSV_NO_BUILD=1
for v in "TSV_AS_SPLIT=1 TSV_AS_S=2" "TSV_AS_SPLIT=1 TSV_AS_S=2 TSV_PRIO=0" "TSV_AS_SPLIT=0 TSV_AS_S=2" "TSV_AS_SPLIT=0 TSV_AS_S=2 TSV_PRIO=0" "TSV_AS_SPLIT=1" "TSV_AS_SPLIT=0"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2f/b.json 2>/dev/null
  echo "$v rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2f/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms'])"
done
