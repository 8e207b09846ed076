set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
for h in 0 1; do
BNF_PLANE=1 BNF_PLANE_L2=1 BNF_PLANE_HINT=$h timeout 300 python scripts/bench_apply.py --configs 3,4 --b 2 > gpurun_out/apply_hint.log 2>&1
python -c "
import json
for l in open('gpurun_out/apply_hint.log'):
    d=json.loads(l); print('hint $h', d['config'], d['b'], round(d['ms_per_apply']*1000,1), {k:v['us'] for k,v in d['passes'].items()})
"
done
BNF_PLANE=1 BNF_PLANE_L2=1 BNF_PLANE_HINT=1 timeout 600 python -m pytest tests -m gpu -x -q -k "middles or plane_l2" > gpurun_out/pytest_hint.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_hint.log
