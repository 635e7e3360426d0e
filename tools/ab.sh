#!/bin/bash
# A/B kernel timing on the same box. Args: label=lib[,ENV=VAL] ...
for spec in "$@"; do
  label=${spec%%=*}; rest=${spec#*=}; lib=${rest%%,*}; envs=""
  [[ "$rest" == *,* ]] && envs=${rest#*,}
  env SPST_LIB=$lib $envs python tools/profile_eval.py > gpurun_out/ab_plain_$label.log 2>&1 || { echo "$label failed"; tail -3 gpurun_out/ab_plain_$label.log; continue; }
  env SPST_LIB=$lib $envs ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/ab_$label.csv python tools/profile_eval.py > /dev/null 2>&1
  env SPST_LIB=$lib $envs python tools/trace_eval.py > gpurun_out/ab_trace_$label.log 2>&1
done
