# per-launch time of the int8 K1 kernels (ncu) at config ${1:-3}
export TSV_K1_OZAKI=${2:-9}
python tools/prof_as.py ${1:-3} > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"oz_|gemm_nt" -c 12 python tools/prof_as.py ${1:-3} 2>/dev/null | grep -v "^==" | awk -F'","' '{n=$5; sub(/\(.*/,"",n); print n, $NF}'
