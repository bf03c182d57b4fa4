# compute-sanitizer memcheck / racecheck / synccheck over small-width kernel tests
set -x
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest -q -m gpu -p no:cacheprovider -x tests/test_ket_gpu.py tests/test_engine_gpu.py \
    "tests/test_executor_gpu.py::test_qft_small_vs_oracle_and_dft" \
    "tests/test_executor_gpu.py::test_random_circuits_golden" \
    "tests/test_executor_gpu.py::test_qft_five_register_bits_vs_oracle" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
