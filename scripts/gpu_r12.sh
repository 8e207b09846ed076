set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
BNF_PLANE=1 BNF_PLANE_L2=1 timeout 900 python -m pytest tests -m gpu -x -q -k "apply_256 or middles or plane_l2" > gpurun_out/pytest_r12.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_r12.log
for e in "BNF_PLANE=1" "BNF_NO_PLANE=1"; do
env $e BNF_PLANE_L2=1 timeout 300 python scripts/bench_apply.py --configs 5 --b 1,2 > gpurun_out/apply_r12.log 2>&1
python -c "
import json
for l in open('gpurun_out/apply_r12.log'):
    d=json.loads(l); print('$e', d['config'], d['b'], round(d['ms_per_apply']*1000,1), {k:v['us'] for k,v in d['passes'].items()})
"
done
