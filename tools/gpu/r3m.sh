out=gpurun_out/r3m
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_schwarz.py tests/test_gpu_symmetry.py tests/test_gpu_parity.py tests/test_online_dt.py tests/test_variants.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $out/pytest.log
for c in 3 4 2; do
for ra in 0 1e-4 1e-6 1e-8; do for m in 1 0.7; do echo "cfg $c replace_at $ra margin $m: $(TSV_REPLACE_AT=$ra TSV_VERIFY_MARGIN=$m python tools/schwarz_perf.py $c | cut -c1-200)"; done; done
done 2>&1 | tee $out/replace.log
