set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python scripts/bench_apply.py --configs 3,4,5 --b 2 > gpurun_out/apply_minb.log 2>&1
python -c "
import json
for l in open('gpurun_out/apply_minb.log'):
    d=json.loads(l); print(d['config'], d['b'], round(d['ms_per_apply']*1000,1), {k:v['us'] for k,v in d['passes'].items()})
"
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_minb.log 2>&1; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_minb.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kpoints_per_s'], d['middle'], d['roofline']['kernel'], d['roofline']['frac'], d['solver']['max_residual']); print({k:v for k,v in d['kernel_ms'].items() if v>1})"
