#!/bin/bash
# ncu --set full of the fused irrep K1 (24 rows per CTA) at config 3
out=gpurun_out/r3d
mkdir -p $out
export TSV_NO_BUILD=1 TSV_SYM_K1_MF=3
python tools/k1_only.py 3 5 > $out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sym_k1_fused -s 2 -c 2 -o $out/k1_fused24 python tools/k1_only.py 3 5 > $out/ncu.log 2>&1
echo "exit $?"; cat $out/plain.log; tail -3 $out/ncu.log
