# The QFT-27 ncu captures behind profiles/ncu_summary.json (bench.py's
# roofline.traffic) plus the bench line of the same build; outputs in gpurun_out/
set -x
out=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qft -s 9 -c 3 -o /tmp/qft_c128 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dropin --no-extra > /dev/null 2>&1
ncu -i /tmp/qft_c128.ncu-rep --page raw --csv > $out/qft27_c128_raw.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qft -s 9 -c 3 -o /tmp/qft_c64 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dropin --no-extra --dtype c64 > /dev/null 2>&1
ncu -i /tmp/qft_c64.ncu-rep --page raw --csv > $out/qft27_c64_raw.csv
