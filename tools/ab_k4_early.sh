# K4 early ticket for mid-range partials: parity, per-CTA timeline, same-box A/B (PRISM_K4_EARLY)
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity_full_size.py tests/test_gpu_concurrency.py tests/test_gpu_paged_op.py -x -q > gpurun_out/kear_tests.log 2>&1; echo rc=$? >> gpurun_out/kear_tests.log
for t in 1 0; do PRISM_K4_EARLY=$t PRISM_K4_PDL=0 FIRST=3584 timeout 200 python tools/k4_cta_trace.py > gpurun_out/kear_cta_$t.txt 2>&1; done
for i in 1 2; do
  for t in 1 0; do
    PRISM_K4_EARLY=$t REPS=3 timeout 300 python tools/k4_bench.py > gpurun_out/kear_${t}_$i.jsonl 2>&1
    PRISM_K4_EARLY=$t REPS=3 CHUNK=2048 timeout 300 python tools/k4_bench.py > gpurun_out/kear2k_${t}_$i.jsonl 2>&1
  done
done
for t in 1 0; do PRISM_K4_EARLY=$t timeout 300 python tools/k4_small.py > gpurun_out/kear_small_$t.jsonl 2>&1; done
