#!/bin/bash
# Schwarz solve timing (configs 3, 4) + per-kernel launch list + Schwarz GPU tests
out=gpurun_out/${1:-ic}; mkdir -p $out
python tools/schwarz_perf.py 3 4 > $out/perf.txt 2>&1
python tools/schwarz_perf.py 3 >> $out/perf.txt 2>&1
bash tools/prof_as_list.sh 3 > $out/list.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "schwarz or parity or golden or configs or variants" > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
