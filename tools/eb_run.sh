cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final2_bench.json 2> /dev/null; tail -c 200 gpurun_out/final2_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/final2_ref.json 2> /dev/null
timeout 900 python bench.py --config c1 > gpurun_out/final2_c1.json 2> /dev/null
timeout 900 python bench.py --config c1 --impl reference > gpurun_out/final2_c1_ref.json 2> /dev/null
timeout 1200 python tools/run_c2_c3.py --out gpurun_out/final2_c2_c3.json > /dev/null 2>&1
timeout 900 python tools/run_c4.py --repeat 2 --out gpurun_out/final2_c4.json > /dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final2_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/final2_*
