# K4 latency-parallel merge: parity tests, then same-box A/B of PRISM_K4_MERGE (tools/k4_bench.py)
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity_full_size.py -x -q > gpurun_out/k4merge_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/k4merge_tests.log
for i in 1 2; do
  for m in 1 0; do
    PRISM_K4_MERGE=$m REPS=3 timeout 300 python tools/k4_bench.py > gpurun_out/k4merge_${m}_$i.jsonl 2> gpurun_out/k4merge_${m}_$i.err
    PRISM_K4_MERGE=$m REPS=3 CHUNK=2048 timeout 300 python tools/k4_bench.py > gpurun_out/k4merge2k_${m}_$i.jsonl 2> gpurun_out/k4merge2k_${m}_$i.err
  done
done
