PRISM_K4_PERM=1 timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q > gpurun_out/s7_tests_perm.log 2>&1; echo rc=$? >> gpurun_out/s7_tests_perm.log
for perm in 0 1; do
  PRISM_K4_PDL=0 PRISM_K4_PERM=$perm FIRST=3584 timeout 200 python tools/k4_cta_trace.py > gpurun_out/k4cta_3584_nopdl_perm$perm.txt 2>&1
  PRISM_K4_PDL=0 PRISM_K4_PERM=$perm FIRST=28160 timeout 200 python tools/k4_cta_trace.py > gpurun_out/k4cta_28160_nopdl_perm$perm.txt 2>&1
done
for perm in 1 0; do PRISM_K4_PERM=$perm REPS=3 timeout 300 python tools/k4_bench.py > gpurun_out/k4perm_$perm.jsonl 2>&1; done
