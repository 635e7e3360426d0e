python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed|FAIL|Error" gpurun_out/gpu_tests.log | tail -5
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json
python tools/coarse_profile.py --dims 756x1008 --m 100 --iters 30 > gpurun_out/coarse1.log 2>&1; grep "ms/iter" gpurun_out/coarse1.log | head -3
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_eval.csv python tools/profile_eval.py > /dev/null 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:conv3x3_tc_kernel --launch-skip 6 -c 1 -o gpurun_out/r02_full_conv128 python tools/profile_eval.py > gpurun_out/ncu1.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:conv3x3_tc_kernel --launch-skip 1 -c 1 -o gpurun_out/r02_full_conv64 python tools/profile_eval.py > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out/*.ncu-rep
