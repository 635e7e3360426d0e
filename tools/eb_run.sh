python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed|FAIL|Error" gpurun_out/gpu_tests.log | tail -5
for lib in paper_2212_13459_b200/libspst.so build/libspst_epi8.so; do
  n=$(basename $lib .so)
  SPST_LIB=$PWD/$lib ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$n.csv python tools/profile_eval.py > /dev/null 2>&1
  SPST_LIB=$PWD/$lib python tools/eval_time.py > gpurun_out/eval_$n.log 2>&1; tail -2 gpurun_out/eval_$n.log
done
