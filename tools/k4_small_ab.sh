for p in 1 0; do PRISM_K4_PDL=$p timeout 300 python tools/k4_small.py > gpurun_out/k4small_pdl$p.jsonl 2>&1; done
CHUNK=512 CTX=512 timeout 300 python tools/k4_trace.py > gpurun_out/k4trace_512.txt 2>&1
CHUNK=512 CTX=4096 timeout 300 python tools/k4_trace.py > gpurun_out/k4trace_512_4k.txt 2>&1
