out=gpurun_out/r3z
mkdir -p $out
export TSV_NO_BUILD=1
echo "base: $(python tools/k1_only.py 3 20) cfg4 $(python tools/k1_only.py 4 20)" | tee $out/bf.log
for v in bfA bfB bfC; do echo "$v: $(TSV_B200_LIB=$PWD/paper_2411_12690_b200/_lib/variants/libtsv_$v.so python tools/k1_only.py 3 20) cfg4 $(TSV_B200_LIB=$PWD/paper_2411_12690_b200/_lib/variants/libtsv_$v.so python tools/k1_only.py 4 20)"; done 2>&1 | tee -a $out/bf.log
