# round 2: full GPU suite (incl. the new cfg2-4 parity) + CPU model check
mkdir -p gpurun_out/r2b
export TSV_NO_BUILD=1
timeout 2400 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider --durations=25 > gpurun_out/r2b/pytest.log 2>&1
echo "pytest_rc=$?"
tail -5 gpurun_out/r2b/pytest.log
timeout 900 python tools/cpu_model_check.py --out gpurun_out/r2b/cpu_model_check_cfg2.json > gpurun_out/r2b/cpu_check.log 2>&1
echo "cpu_check_rc=$?"
