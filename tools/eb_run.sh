python -m pytest tests -m gpu -q -x -s > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed|FAIL|Error" gpurun_out/gpu_tests.log | tail -5
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 800 gpurun_out/bench_ref.json
python bench.py --config c1 --steps 10 --warmup 0 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -c 900 gpurun_out/bench_c1.json
python bench.py --impl reference --config c1 --steps 10 --warmup 0 > gpurun_out/bench_c1_ref.json 2> gpurun_out/bench_c1_ref.err; tail -c 900 gpurun_out/bench_c1_ref.json
