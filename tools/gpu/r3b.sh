#!/bin/bash
out=gpurun_out/r3b
mkdir -p $out
export TSV_NO_BUILD=1
timeout 900 python tools/sym_probe.py 3 400 > $out/probe3.log 2>&1; echo "exit $?"; cat $out/probe3.log | cut -c1-1500
