# full GPU suite + default bench (cfg3) + cfg4/cfg2 bench lines
mkdir -p gpurun_out/r2g
export TSV_NO_BUILD=1
timeout 2700 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider --durations=30 > gpurun_out/r2g/pytest.log 2>&1
echo "pytest_rc=$?"; tail -3 gpurun_out/r2g/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2g/bench_cfg3.json 2> gpurun_out/r2g/bench_cfg3.err
echo "bench3 rc=$?"
for c in 4 2 1 0; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g/bench_cfg$c.json 2> gpurun_out/r2g/bench_cfg$c.err
echo "bench$c rc=$?"
done
