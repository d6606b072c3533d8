out=gpurun_out/r3x
mkdir -p $out
export TSV_NO_BUILD=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_symmetry.py tests/test_variants.py tests/test_cutplane.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $out/pytest.log
