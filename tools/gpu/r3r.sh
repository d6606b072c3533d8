out=gpurun_out/r3r
mkdir -p $out
export TSV_NO_BUILD=1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --log-file $out/racecheck.log python -m pytest tests/test_gpu_symmetry.py -m gpu -x -q -p no:cacheprovider -k "operator" > $out/race_pytest.log 2>&1; echo "racecheck exit $?"; tail -3 $out/race_pytest.log; tail -8 $out/racecheck.log
