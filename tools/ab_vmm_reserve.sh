# Same-box A/B of the VMM handle reserve knobs on the C2 churn stress loop
# (tools/vmm_churn_repeat.py, 3 in-process runs per configuration).
set -x
run() { tag=$1; shift; env "$@" REPS=3 timeout 300 python tools/vmm_churn_repeat.py > gpurun_out/ab2_$tag.jsonl 2> gpurun_out/ab2_$tag.err; echo "$tag rc=$?"; }
run D1 PRISM_VMM_RESERVE_CHUNKS=8
run A1 PRISM_VMM_RESERVE_CHUNKS=0
run E1 PRISM_VMM_RESERVE_CHUNKS=16
run F1 PRISM_VMM_RESERVE_CHUNKS=8 PRISM_VMM_RESERVE_BATCH=4
run D2 PRISM_VMM_RESERVE_CHUNKS=8
run A2 PRISM_VMM_RESERVE_CHUNKS=0
run E2 PRISM_VMM_RESERVE_CHUNKS=16
run F2 PRISM_VMM_RESERVE_CHUNKS=8 PRISM_VMM_RESERVE_BATCH=4
run D3 PRISM_VMM_RESERVE_CHUNKS=8
run A3 PRISM_VMM_RESERVE_CHUNKS=0
