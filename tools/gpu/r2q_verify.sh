mkdir -p gpurun_out/r2q
export TSV_NO_BUILD=1
b() { env $1 timeout 600 python bench.py --config $2 --steps $3 --warmup 5 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2q/b.json 2>gpurun_out/r2q/b.err; echo "cfg$2 $1 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2q/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms']['per_iteration'])" || tail -5 gpurun_out/r2q/b.err; }
for c in 0 1 2; do b "TSV_K1_VERIFY=0" $c 200; b "TSV_K1_VERIFY=10" $c 200; done
b "TSV_K1_VERIFY=0" 3 5; b "TSV_K1_VERIFY=0" 4 5
