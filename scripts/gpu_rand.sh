set -x
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 400 python scripts/tune_qft.py 30 c64 rand > gpurun_out/tune_rand_c64.log 2>&1
timeout 400 python scripts/tune_qft.py 30 c128 rand > gpurun_out/tune_rand_c128.log 2>&1
timeout 300 python scripts/tune_qft.py 27 c64 > gpurun_out/tune_c64.log 2>&1
cat gpurun_out/tune_rand_c64.log gpurun_out/tune_rand_c128.log gpurun_out/tune_c64.log
