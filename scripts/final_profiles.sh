# Round-end evidence on one B200 (run via gpurun); outputs land in gpurun_out/
# and are summarised into profiles/ afterwards (scripts/make_ncu_summary.py,
# scripts/pergate_table.py).
set -x
out=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > $out/gpu_tests.txt
timeout 600 python bench.py 2>&1 | tail -1 > $out/bench.json
timeout 600 python bench.py --impl reference 2>&1 | tail -1 > $out/bench_reference.json
# launch list of the bench (cold, serialised: shares, not absolutes)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-dropin --no-extra > /dev/null 2>&1
# full captures of the QFT-27 sweeps, c128 (headline) and c64
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qft -s 9 -c 3 -o /tmp/qft_c128 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dropin --no-extra > /dev/null 2>&1
ncu -i /tmp/qft_c128.ncu-rep --page raw --csv > $out/qft27_c128_raw.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qft -s 9 -c 3 -o /tmp/qft_c64 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dropin --no-extra --dtype c64 > /dev/null 2>&1
ncu -i /tmp/qft_c64.ncu-rep --page raw --csv > $out/qft27_c64_raw.csv
# per-gate kernels at w = 28 / 27
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/pergate_c64.csv python scripts/pergate_bw.py 28 c64 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/pergate_c128.csv python scripts/pergate_bw.py 27 c128 > /dev/null 2>&1
# one generic sweep of random 30x20 c64 (k_sweep LEAN)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 4 -c 1 -o /tmp/ks -f \
  python scripts/prof_rand.py 30 c64 > /dev/null 2>&1
ncu -i /tmp/ks.ncu-rep --page raw --csv > $out/ks_raw.csv
# sanitizers over the generic-sweep opcode tests
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest -q -m gpu -p no:cacheprovider tests/test_sweep_opcodes_gpu.py -k couplers_only > $out/sanitize_sweep_$tool.log 2>&1
  echo "$tool rc=$?" >> $out/sanitize_sweep.txt
done
# the other BASELINE configs and the engine
timeout 1200 python scripts/bench_configs.py qft20 qft27 rand30 qft34 hybrid > $out/configs.jsonl 2>&1
timeout 600 python scripts/engine_profile.py 5 > $out/engine.txt 2>&1
timeout 600 python scripts/engine_phases.py >> $out/engine.txt 2>&1
ls -la $out
