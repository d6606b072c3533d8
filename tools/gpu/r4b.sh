out=gpurun_out/r4b
mkdir -p $out
export TSV_NO_BUILD=1
for c in 3 4 2; do for w in 1 0; do echo "cfg$c wave $w: $(TSV_VEC_WAVE=$w python tools/schwarz_perf.py $c | cut -c1-200)"; done; done | tee $out/wave.log
