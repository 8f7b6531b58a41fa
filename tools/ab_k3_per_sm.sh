# K3 shape-aware CTAs per SM: parity, then same-box A/B on the 8 SURVEY shapes (PRISM_SK_PER_SM_AUTO)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/k3auto_tests.log 2>&1; echo rc=$? >> gpurun_out/k3auto_tests.log
for i in 1 2; do
  for a in 1 0; do PRISM_SK_PER_SM_AUTO=$a timeout 200 python tools/k3_shapes.py > gpurun_out/k3auto_${a}_$i.jsonl 2>&1; done
done
for a in 1 0; do PRISM_SK_PER_SM_AUTO=$a timeout 300 python bench.py --no-churn --no-prefill --no-slo --no-serving --no-cpu-baseline > gpurun_out/k3auto_bench_$a.json 2>/dev/null; done
