export TSV_NO_BUILD=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke exit $?"
timeout 600 python -m pytest tests/test_gpu_symmetry.py tests/test_schwarz.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-jacobi-leg --e2e-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['gpu_launches'], d['roofline']['frac'])"
