#!/bin/bash
out=gpurun_out/r3h
mkdir -p $out
export TSV_NO_BUILD=1 TSV_SYM_STAGGER_NS=0
for v in A B C D E F; do for mf in 2 3; do for ab in 0 1 2; do
echo "variant $v mf $mf ablate $ab: $(TSV_B200_LIB=$PWD/paper_2411_12690_b200/_lib/variants/libtsv_sym$v.so TSV_SYM_K1_MF=$mf TSV_SYM_ABLATE=$ab python tools/k1_only.py 3 20)"; done; done; done 2>&1 | tee $out/variants.log
