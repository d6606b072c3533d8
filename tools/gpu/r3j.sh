# full GPU suite with the fused irrep K1 default
out=gpurun_out/r3j
mkdir -p $out
export TSV_NO_BUILD=1
timeout 3000 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=15 > $out/pytest.log 2>&1
echo "pytest_rc=$?"; tail -30 $out/pytest.log
