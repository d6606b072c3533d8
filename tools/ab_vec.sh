mkdir -p gpurun_out/ab1
for v in old u1 default; do
  if [ $v = default ]; then unset TSV_B200_LIB; else export TSV_B200_LIB=$PWD/paper_2411_12690_b200/_lib/variants/libtsv_$v.so; fi
  echo "== $v" >> gpurun_out/ab1/perf.txt
  python tools/schwarz_perf.py 3 >> gpurun_out/ab1/perf.txt 2>&1
  python tools/schwarz_perf.py 3 >> gpurun_out/ab1/perf.txt 2>&1
  bash tools/prof_as_list.sh 3 > gpurun_out/ab1/list_$v.txt 2>&1
done
