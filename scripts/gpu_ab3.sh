set -x
timeout 600 python -m pytest tests/test_executor_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for v in 1 0; do SK_QFT_VSTORE=$v timeout 300 python scripts/tune_qft.py 27 c64 > gpurun_out/tune_c64_v$v.log 2>&1; done
cat gpurun_out/tune_c64_v*.log
