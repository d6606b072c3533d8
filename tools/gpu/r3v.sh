out=gpurun_out/r3v
mkdir -p $out
export TSV_NO_BUILD=1
timeout 1800 python -m pytest tests/test_gpu_configs.py tests/test_gpu_symmetry.py tests/test_schwarz.py tests/test_variants.py -m gpu -x -q -s -p no:cacheprovider -k "not large_config" > $out/pytest.log 2>&1; echo "pytest exit $?"; grep "cfg2\|passed\|failed" $out/pytest.log | cut -c1-300
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_cfg2.json 2> $out/bench_cfg2.err; python -c "
import json
d=json.loads(open('$out/bench_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', d['value'], d['ms_per_step'], d['phase_ms'], d['config']['iterations'], d['roofline']['kernel'][:30], d['roofline']['frac'])"
