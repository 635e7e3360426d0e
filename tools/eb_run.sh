python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_f1b2.json 2> gpurun_out/bench_f1b2.err; tail -c 600 gpurun_out/bench_f1b2.json
SPST_BWD_DRAIN=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f1b1.json 2>&1; tail -c 300 gpurun_out/bench_f1b1.json
SPST_FWD_DRAIN=2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f2b2.json 2>&1; tail -c 300 gpurun_out/bench_f2b2.json
SPST_BWD_DRAIN=1 python tools/error_budget.py --out gpurun_out/eb_f1b1c.json > gpurun_out/eb_f1b1c.log 2>&1
python tools/error_budget.py --out gpurun_out/eb_f1b2c.json > gpurun_out/eb_f1b2c.log 2>&1
python tools/rz_calibrate.py > gpurun_out/rz_default.json 2>&1
