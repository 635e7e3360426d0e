for lib in build/libspst_base.so paper_2212_13459_b200/libspst.so build/libspst_base.so paper_2212_13459_b200/libspst.so; do
  SPST_LIB=$PWD/$lib python tools/eval_time.py 2>&1 | tail -1
done
for lib in build/libspst_base.so paper_2212_13459_b200/libspst.so; do
  n=$(basename $lib .so)
  SPST_LIB=$PWD/$lib ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$n.csv python tools/profile_eval.py > /dev/null 2>&1
done
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_maxpool.py tests/test_gpu_parity.py -q -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
