# K4 PDL chain: parity tests, then same-box A/B of PRISM_K4_PDL (tools/k4_bench.py, 512-token chunks)
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity_full_size.py tests/test_gpu_concurrency.py -x -q > gpurun_out/k4pdl_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/k4pdl_tests.log
for i in 1 2; do
  for p in 1 0; do
    PRISM_K4_PDL=$p REPS=3 timeout 300 python tools/k4_bench.py > gpurun_out/k4pdl_${p}_$i.jsonl 2> gpurun_out/k4pdl_${p}_$i.err
  done
done
