#!/bin/bash
# Round-2 (third session) evidence pass on one B200 with the irrep K1 / K6 path and the
# residual-replacement Schwarz loop: GPU tests, smoke, both bench arms at config 3, bench
# lines for configs 0-4, the ncu launch list of the bench command, and full ncu captures
# of the iteration kernels (incl. sym_k1_fused_kernel) and the recovery kernels.
tag=${1:-r3_final}
out=gpurun_out/$tag
mkdir -p $out
export TSV_NO_BUILD=1
nvidia-smi > $out/nvidia-smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 2700 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider --durations=20 > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" | tee -a $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" | tee -a $out/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $out/bench_cfg3.json 2> $out/bench_cfg3.err; echo "bench exit $?"
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_ref_cfg3.json 2> $out/bench_ref_cfg3.err; echo "ref exit $?"
for c in 4 2; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_cfg$c.json 2> $out/bench_cfg$c.err; echo "bench$c exit $?"; done
for c in 1 0; do timeout 900 python bench.py --config $c --steps 400 --warmup 10 --no-cpu-baseline > $out/bench_cfg$c.json 2> $out/bench_cfg$c.err; echo "bench$c exit $?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench_cfg3.csv \
  python bench.py --steps 2 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > $out/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:sym_k1_fused|as_scatter|tc_local_pair|as_restrict|as_zl|cg_gather|as_update|as_coarse' --launch-skip 60 --launch-count 12 \
  -o $out/iter_kernels_full python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > $out/ncu_iter.log 2>&1; echo "ncu iter exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:stress_kernel|k6_face|gemm_seg|sym_fine' -c 4 \
  -o $out/recovery_full python bench.py --steps 1 --warmup 1 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > $out/ncu_rec.log 2>&1; echo "ncu rec exit $?"
python tools/launch_shares.py $out/launches_bench_cfg3.csv > $out/launch_shares_bench_cfg3.csv 2>/dev/null
python tools/ncu_hbm_table.py $out/iter_kernels_full.ncu-rep --config 3 --bench-json $out/bench_cfg3.json > $out/iter_kernels_cfg3.csv 2>/dev/null
gzip -f $out/launches_bench_cfg3.csv
