#!/bin/bash
# Fused irrep K1: parity tests, then config-3 probe of the variants
out=gpurun_out/r3c
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_symmetry.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -15 $out/pytest.log
timeout 1500 python tools/sym_probe.py 3 400 > $out/probe3.log 2>&1; echo "exit $?"; cut -c1-600 $out/probe3.log
