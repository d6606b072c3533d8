set -x
nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out/r2a
timeout 600 python bench.py --steps 2 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
echo bench_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:as_scatter|tc_local_pair|as_restrict|as_zl|cg_gather|as_update|as_coarse' --launch-skip 40 --launch-count 9 -o gpurun_out/r2a/hbm_kernels python bench.py --steps 1 --warmup 3 --no-jacobi-leg --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2a/ncu.log 2>&1
echo ncu_rc=$?
