# A/B: QFT tile geometries with the dedicated k_qft kernel vs the generic k_sweep
set -x
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for k in 1 0; do
SK_QFT_KERNEL=$k timeout 300 python scripts/tune_qft.py 27 c64 > gpurun_out/tune_c64_k$k.log 2>&1
SK_QFT_KERNEL=$k timeout 300 python scripts/tune_qft.py 27 c128 > gpurun_out/tune_c128_k$k.log 2>&1
done
for f in gpurun_out/tune_*_k*.log; do echo == $f; cat $f; done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
