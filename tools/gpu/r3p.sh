out=gpurun_out/r3p
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_symmetry.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -4 $out/pytest.log
for pipe in 0 1; do for tail in 1 0; do
echo "pipe $pipe tail $tail: $(TSV_SYM_K1_PIPE=$pipe TSV_SYM_K1_TAIL=$tail python tools/k1_only.py 3 20)"; done; done 2>&1 | tee $out/k1.log
echo "cfg4 pipe0: $(python tools/k1_only.py 4 20)"; echo "cfg4 pipe1: $(TSV_SYM_K1_PIPE=1 python tools/k1_only.py 4 20)"
