set -x
for m in 0 1; do
SK_SWEEP_PIPE=$m timeout 300 python scripts/tune_qft.py 27 c64 > gpurun_out/tune_c64_p$m.log 2>&1
SK_SWEEP_PIPE=$m timeout 300 python scripts/tune_qft.py 27 c128 > gpurun_out/tune_c128_p$m.log 2>&1
done
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for f in gpurun_out/tune_*_p*.log; do echo == $f; cat $f; done
