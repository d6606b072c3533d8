out=gpurun_out/r3l
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_symmetry.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $out/pytest.log
for mf in 2 3; do for ab in 0 2; do
echo "mf $mf ablate $ab: $(TSV_SYM_K1_MF=$mf TSV_SYM_ABLATE=$ab python tools/k1_only.py 3 20)"; done; done 2>&1 | tee $out/k1.log
