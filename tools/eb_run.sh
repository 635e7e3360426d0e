cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_split.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench_split.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['clocks'],d['roofline']['classes'])"
