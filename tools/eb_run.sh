python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed|FAIL|Error" gpurun_out/gpu_tests.log | tail -5
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json
python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -c 300 gpurun_out/bench_c1.json
python bench.py --impl reference --config c1 --steps 10 --warmup 0 > gpurun_out/bench_c1_ref.json 2> gpurun_out/bench_c1_ref.err; tail -c 300 gpurun_out/bench_c1_ref.json
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -o gpurun_out/r02_dram python tools/profile_eval.py > gpurun_out/ncu_dram.log 2>&1
python tools/ncu_traffic.py gpurun_out/r02_dram.ncu-rep "conv3x3_tc_kernel<128" "conv3x3_tc<128>" > gpurun_out/dominant_traffic.json; cat gpurun_out/dominant_traffic.json
python tools/run_c4.py --out gpurun_out/c4_fast.json > gpurun_out/c4_fast.log 2>&1; python -c "
import json; d=json.load(open('gpurun_out/c4_fast.json')); print(d['total_seconds'], [(s['scale'], round(s['ms_per_iter'],2), round(s['seconds'],2)) for s in d['scales']])"
