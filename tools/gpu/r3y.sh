out=gpurun_out/r3y
mkdir -p $out
export TSV_NO_BUILD=1
for c in 3 4; do echo "cfg$c: $(python tools/schwarz_perf.py $c | cut -c1-230)"; done | tee $out/perf.log
timeout 900 python -m pytest tests/test_schwarz.py tests/test_gpu_parity.py tests/test_online_dt.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest.log
