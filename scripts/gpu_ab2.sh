set -x
timeout 600 python -m pytest tests/test_executor_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/tune_qft.py 27 c64 > gpurun_out/tune_c64.log 2>&1
timeout 300 python scripts/tune_qft.py 27 c128 > gpurun_out/tune_c128.log 2>&1
cat gpurun_out/tune_c64.log gpurun_out/tune_c128.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qft -s 9 -c 3 -o gpurun_out/prof -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu2.log 2>&1
