out=gpurun_out/r3s
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-jacobi-leg --e2e-steps 0 > $out/bench_cfg3.json 2> $out/bench_cfg3.err; echo "bench exit $?"
python -c "
import json
d=json.loads(open('$out/bench_cfg3.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step']); print(json.dumps(d['roofline'])); print(json.dumps(d['roofline_other']))"
timeout 600 python -m pytest tests/test_abi.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
