# full GPU suite + default bench (cfg3) + other configs, with the fused irrep K1 default
out=gpurun_out/r3i
mkdir -p $out
export TSV_NO_BUILD=1
timeout 2700 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider --durations=15 > $out/pytest.log 2>&1
echo "pytest_rc=$?"; tail -25 $out/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench_cfg3.json 2> $out/bench_cfg3.err
echo "bench3 rc=$?"; cut -c1-1500 $out/bench_cfg3.json
for c in 4 2; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_cfg$c.json 2> $out/bench_cfg$c.err
echo "bench$c rc=$?"; cut -c1-700 $out/bench_cfg$c.json
done
