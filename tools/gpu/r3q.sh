out=gpurun_out/r3q
mkdir -p $out
export TSV_NO_BUILD=1
for c in 3 4 2; do for ov in 1 0; do echo "cfg $c overlap $ov: $(TSV_REC_OVERLAP=$ov python tools/rec_ab.py $c)"; done; done 2>&1 | tee $out/rec.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_schwarz.py -m gpu -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $out/pytest.log
