for b in 16 24 32 48; do for p in 0 1 2; do
  if [ $p = 0 ]; then e=""; else e="PRISM_SK_PER_SM=$p"; fi
  env $e B=$b SHAPES=llama3.1-8b,llama3.2-1b timeout 120 python tools/k3_shapes.py | sed "s/^/{\"B\": $b, \"pps\": $p, \"r\": /; s/$/}/" >> gpurun_out/k3x.jsonl 2>/dev/null
done; done
for b in 96 128 192; do for p in 0 1 2; do
  if [ $p = 0 ]; then e=""; else e="PRISM_SK_PER_SM=$p"; fi
  env $e B=$b SHAPES=qwen2.5-7b,qwen2.5-1.5b,qwen2.5-0.5b timeout 120 python tools/k3_shapes.py | sed "s/^/{\"B\": $b, \"pps\": $p, \"r\": /; s/$/}/" >> gpurun_out/k3x.jsonl 2>/dev/null
done; done
