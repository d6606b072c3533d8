#!/bin/bash
# One GPU-box pass: tests, smoke, bench (both arms), launch list of the bench command.
# Usage: tools/gpu_round.sh [tag]   (outputs under gpurun_out/<tag>/)
tag=${1:-r1}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench exit $?" >> $out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > $out/ncu_bench.log 2>&1
echo "ncu exit $?" >> $out/ncu_bench.log
# full ncu captures of the dominant kernels (K1 operator apply, K7 stress)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_nt_f64 --launch-skip 3 -c 1 \
  -o $out/k1_full python tools/prof_as.py 3 > $out/ncu_k1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stress_kernel -c 1 \
  -o $out/k7_full python tools/prof_recover.py 3 > $out/ncu_k7.log 2>&1
