#!/bin/bash
out=gpurun_out/${1:-pdl}; mkdir -p $out
python tools/schwarz_perf.py 3 4 > $out/pdl.txt 2>&1
TSV_NO_PDL=1 python tools/schwarz_perf.py 3 4 > $out/nopdl.txt 2>&1
python tools/schwarz_perf.py 3 >> $out/pdl.txt 2>&1
TSV_NO_PDL=1 python tools/schwarz_perf.py 3 >> $out/nopdl.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
