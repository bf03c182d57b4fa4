set -x
bash scripts/gpu_check.sh
timeout 300 python scripts/tune_qft.py 27 c64 > gpurun_out/tune_c64.log 2>&1
timeout 300 python scripts/tune_qft.py 27 c128 > gpurun_out/tune_c128.log 2>&1
cat gpurun_out/tune_c64.log gpurun_out/tune_c128.log
