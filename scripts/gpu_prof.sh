# ncu: launch list of the bench + a full capture of the k_qft sweeps
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qft -s 9 -c 3 -o gpurun_out/prof -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
