#!/bin/bash
out=gpurun_out/r3e
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_symmetry.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -5 $out/pytest.log
timeout 1500 python tools/sym_probe.py 3 400 fused16 fused24 > $out/probe3.log 2>&1; echo "exit $?"; cut -c1-600 $out/probe3.log
