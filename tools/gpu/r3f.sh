#!/bin/bash
# ncu --set full of the fused irrep K1 (16 rows per CTA, 2 CTAs per SM) at config 3
out=gpurun_out/r3f
mkdir -p $out
export TSV_NO_BUILD=1
python tools/k1_only.py 3 5 > $out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sym_k1_fused -s 2 -c 1 -o $out/k1_fused16 python tools/k1_only.py 3 5 > $out/ncu.log 2>&1
echo "exit $?"; cat $out/plain.log; tail -2 $out/ncu.log
