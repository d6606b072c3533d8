out=gpurun_out/r3w
mkdir -p $out
export TSV_NO_BUILD=1
for u in 1 2 4; do echo "fine unroll $u cfg3: $(TSV_B200_LIB=$PWD/paper_2411_12690_b200/_lib/variants/libtsv_fine$u.so python tools/rec_ab.py 3)"; done 2>&1 | tee $out/fine.log
echo "fine unroll 4 cfg4: $(TSV_B200_LIB=$PWD/paper_2411_12690_b200/_lib/variants/libtsv_fine4.so python tools/rec_ab.py 4)" | tee -a $out/fine.log
