# launch list of one Schwarz solve + recovery at config 3 (fused irrep K1)
out=gpurun_out/r3k
mkdir -p $out
export TSV_NO_BUILD=1
python tools/schwarz_perf.py 3 > $out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/schwarz_perf.py 3 > $out/ncu.log 2>&1
echo "ncu exit $?"; cat $out/plain.log
python tools/launch_summary.py $out/launches.csv > $out/launch_summary.txt 2>&1; head -50 $out/launch_summary.txt
gzip -f $out/launches.csv
