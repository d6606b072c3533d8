out=gpurun_out/r3o
mkdir -p $out
export TSV_NO_BUILD=1
for mf in 2 1; do for ab in 0 1 2; do
echo "mf $mf ablate $ab: $(TSV_SYM_K1_MF=$mf TSV_SYM_ABLATE=$ab python tools/k1_only.py 3 20)"; done; done 2>&1 | tee $out/k1.log
TSV_SYM_K1=1 TSV_SYM_K1_MF=1 timeout 600 python -m pytest tests/test_gpu_symmetry.py -m gpu -x -q -p no:cacheprovider -k "fused16 and operator" 2>&1 | tail -3
