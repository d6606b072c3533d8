out=gpurun_out/r4c
mkdir -p $out
export TSV_NO_BUILD=1
echo "base cfg3: $(python tools/schwarz_perf.py 3 | cut -c1-200)" | tee $out/rw.log
for w in 4 2; do for c in 3 4; do echo "rw$w cfg$c: $(TSV_B200_LIB=$PWD/paper_2411_12690_b200/_lib/variants/libtsv_rw$w.so python tools/schwarz_perf.py $c | cut -c1-200)"; done; done | tee -a $out/rw.log
