cd $GRAFT_REPO_ROOT
timeout 300 python tools/coarse_profile.py 2>&1 | grep -v Warning | tail -45 > gpurun_out/coarse_host2.log
timeout 600 python tools/run_c4.py --repeat 2 --out gpurun_out/c4_host2.json > /dev/null 2>&1
python -c "
import json;d=json.load(open('gpurun_out/c4_host2.json'))
for r in d['runs']: print(r['kind'], round(r['total_seconds'],2), [(s['scale'], round(s['ms_per_iter'],2), round(s['seconds'],2)) for s in r['scales']])"
