out=gpurun_out/r3u
mkdir -p $out
export TSV_NO_BUILD=1
for c in 2 1; do
echo "cfg$c default: $(python tools/k1_only.py $c 50)"
echo "cfg$c irrep16: $(TSV_SYM_K1=1 python tools/k1_only.py $c 50)"
echo "cfg$c irrep24: $(TSV_SYM_K1=1 TSV_SYM_K1_MF=3 python tools/k1_only.py $c 50)"
done 2>&1 | tee $out/k1_small.log
