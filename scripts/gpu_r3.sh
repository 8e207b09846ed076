set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r3.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_r3.log
for cfg in "BNF_PLANE=1" "BNF_NO_PLANE=1"; do
  echo "== $cfg"
  env $cfg timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 2 > gpurun_out/apply_r3.log 2>&1
  python -c "
import json
for l in open('gpurun_out/apply_r3.log'):
    d=json.loads(l); print(d['config'], d['b'], round(d['ms_per_apply']*1000,1), {k:v['us'] for k,v in d['passes'].items()})
"
done
timeout 900 python bench.py > gpurun_out/bench_r3.log 2>&1; echo bench rc=$?
cut -c1-3000 gpurun_out/bench_r3.log
timeout 900 python bench.py --warm 0 --no-cpu --no-e2e > gpurun_out/bench_r3cold.log 2>&1; echo bench rc=$?
cut -c1-600 gpurun_out/bench_r3cold.log
