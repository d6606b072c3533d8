#!/bin/bash
# Round 3 probe: mirror-symmetric K1/K6 path — parity tests, config-3 timing with the path on/off, launch list.
out=gpurun_out/r3a
mkdir -p $out
export TSV_NO_BUILD=1
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_symmetry.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_schwarz.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?" | tee -a $out/pytest.log
tail -5 $out/pytest.log
TSV_TIMING=1 timeout 600 python tools/schwarz_perf.py 3 > $out/perf_sym.log 2> $out/perf_sym.err; echo "sym exit $?"; cat $out/perf_sym.log; grep -i "symmetry" $out/perf_sym.err
TSV_SYM_K1=0 timeout 600 python tools/schwarz_perf.py 3 > $out/perf_k6only.log 2>&1; echo "k6only exit $?"; cat $out/perf_k6only.log
TSV_SYM=0 timeout 600 python tools/schwarz_perf.py 3 > $out/perf_plain.log 2>&1; echo "plain exit $?"; cat $out/perf_plain.log
TSV_SYM_CORR=0 timeout 600 python tools/schwarz_perf.py 3 > $out/perf_nocorr.log 2>&1; echo "nocorr exit $?"; cat $out/perf_nocorr.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/schwarz_perf.py 3 > $out/ncu.log 2>&1; echo "ncu exit $?"
python tools/launch_summary.py $out/launches.csv > $out/launch_summary.txt 2>&1; head -40 $out/launch_summary.txt
