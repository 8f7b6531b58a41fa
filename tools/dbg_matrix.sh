T="timeout 400"
$T python -m pytest tests/test_gpu_vmm.py -q -x > gpurun_out/r_test.log 2>&1
PRISM_SERVE_SYNC=1 $T python tools/debug_serving.py c5 6 120 1 1 > gpurun_out/r_sync1.log 2>&1
$T python tools/debug_serving.py c5 6 120 1 1 > gpurun_out/r_nosync1.log 2>&1
$T python tools/debug_serving.py c5 6 120 1 0 > gpurun_out/r_nosync0.log 2>&1
