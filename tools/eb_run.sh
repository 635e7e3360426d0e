SPST_DEBUG_RANGES=1 python tools/repro_switch.py > gpurun_out/repro.log 2>&1; grep -v "careful 0: amax" gpurun_out/repro.log | tail -30
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed|Error|FAIL" gpurun_out/gpu_tests.log | tail -8
