set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
for cw in 16 32 64; do
BNF_PLANE=1 BNF_PLANE_L2=1 BNF_PLANE_CW=$cw timeout 300 python scripts/bench_apply.py --configs 4 --b 2 > gpurun_out/apply_l2cw.log 2>&1
python -c "
import json
for l in open('gpurun_out/apply_l2cw.log'):
    d=json.loads(l); print('cw $cw', d['config'], d['b'], round(d['ms_per_apply']*1000,1), {k:v['us'] for k,v in d['passes'].items()})
"
done
BNF_PLANE=1 BNF_PLANE_L2=1 BNF_PLANE_CW=64 timeout 600 python -m pytest tests -m gpu -x -q -k "apply_vs_matrixfree" > gpurun_out/pytest_l2cw.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_l2cw.log
