python -m pytest tests/test_gpu_contracts.py tests/test_gpu_kernels.py -q -x -s > gpurun_out/t.log 2>&1; grep -E "fp16|passed|failed|Error" gpurun_out/t.log | tail -5
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision fp16 > gpurun_out/bench_fp16.json 2> gpurun_out/bench_fp16.err; tail -c 300 gpurun_out/bench_fp16.json
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json
