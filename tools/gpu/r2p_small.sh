mkdir -p gpurun_out/r2p
export TSV_NO_BUILD=1
b() { env $1 timeout 600 python bench.py --config $2 --steps $3 --warmup 5 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2p/b.json 2>gpurun_out/r2p/b.err; echo "cfg$2 $1 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2p/b.json').read().strip().splitlines()[-1]);c=d['config'];print(d['value'],c['iterations'],c['restarts'],d['phase_ms']['per_iteration'])" || tail -5 gpurun_out/r2p/b.err; }
for n in 148 74 32 16; do for c in 0 1; do b "TSV_SMALL_PCG=1 TSV_SMALL_PCG_CTAS=$n" $c 300; done; done
