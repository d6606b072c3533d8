out=gpurun_out/r4a
mkdir -p $out
export TSV_NO_BUILD=1
for c in 3 4; do for sv in 0 1; do echo "cfg$c serial $sv: $(TSV_AS_SERIAL=$sv python tools/schwarz_perf.py $c | cut -c1-200)"; done; done | tee $out/serial.log
