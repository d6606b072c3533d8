out=gpurun_out/r3t
mkdir -p $out
export TSV_NO_BUILD=1
for mf in 2 3 4; do echo "cfg4 mf $mf: $(TSV_SYM_K1_MF=$mf python tools/k1_only.py 4 20)"; done 2>&1 | tee $out/k1_cfg4.log
for ab in 1 2 4 6; do echo "cfg4 mf 2 ablate $ab: $(TSV_SYM_ABLATE=$ab python tools/k1_only.py 4 20)"; done 2>&1 | tee -a $out/k1_cfg4.log
