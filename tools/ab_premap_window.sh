# Look-ahead window depth (PRISM_PREMAP_PAGES 256 vs the earlier 128), same box: C1 + scheduler-driven serving
for i in 1 2; do for w in 256 128; do
  PRISM_PREMAP_PAGES=$w timeout 400 python bench.py --no-churn --no-prefill --no-slo --no-cpu-baseline > gpurun_out/win_${w}_$i.json 2>/dev/null
done; done
