cd $GRAFT_REPO_ROOT
for lib in build/libspst_old.so paper_2212_13459_b200/libspst.so build/libspst_old.so paper_2212_13459_b200/libspst.so; do SPST_LIB=$PWD/$lib timeout 300 python tools/eval_time.py | tail -1; done
for lib in build/libspst_old.so paper_2212_13459_b200/libspst.so; do n=$(basename $lib .so); SPST_LIB=$PWD/$lib timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$n.csv python tools/profile_eval.py > /dev/null 2>&1; done
