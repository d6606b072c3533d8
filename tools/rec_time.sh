#!/bin/bash
# Recovery timing (K6 GEMM + K7 stress) at configs 3 and 4, plus per-kernel ncu durations.
out=gpurun_out/${1:-rec}
mkdir -p $out
for c in 3 4; do REPS=4 python tools/prof_recover.py $c > $out/rec_cfg$c.txt 2>&1; done
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"stress|gemm_nt" \
  python tools/prof_recover.py 3 2>/dev/null | grep -v "^==" > $out/rec_ncu_cfg3.csv
