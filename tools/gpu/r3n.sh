out=gpurun_out/r3n
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_schwarz.py tests/test_abi.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -12 $out/pytest.log
