export TSV_K1_OZAKI=9
python tools/prof_as.py 3 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:"oz_" -c 6 python tools/prof_as.py 3 2>/dev/null | grep -v "^==" 
