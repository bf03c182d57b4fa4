# one gpurun call: GPU tests, smoke, bench, ncu launch list + full capture of the top kernel
# (the .ncu-rep stays in /tmp on the box; its raw CSV comes back in gpurun_out/)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qft -s 9 -c 3 -o /tmp/prof -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu2.log 2>&1
ncu -i /tmp/prof.ncu-rep --page raw --csv > gpurun_out/prof_raw.csv
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_src.csv
ls -la gpurun_out
