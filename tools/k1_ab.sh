#!/bin/bash
# K1 dynamic tile queue vs forced stream-K (configs 3, 4), and the set-up phase timings
out=gpurun_out/${1:-k1ab}; mkdir -p $out
python tools/quick_perf.py 3 4 > $out/dyn.txt 2>&1
TSV_STREAMK=1 python tools/quick_perf.py 3 4 > $out/sk.txt 2>&1
python tools/schwarz_perf.py 3 > $out/perf_dyn.txt 2>&1
TSV_STREAMK=1 python tools/schwarz_perf.py 3 > $out/perf_sk.txt 2>&1
TSV_TIMING=1 python tools/setup_debug.py 3 > $out/setup3.txt 2>&1
TSV_TIMING=1 python tools/e2e_breakdown.py 3 > $out/e2e3.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "schwarz or parity or golden or configs" > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
