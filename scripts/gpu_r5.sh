set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r5.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke_r5.log
for cfg in "BNF_Z_UNROLL=1" "BNF_Z_UNROLL=2"; do
  echo "== $cfg"
  env $cfg BNF_NO_PLANE=1 timeout 300 python scripts/bench_apply.py --configs 3,4 --b 2 > gpurun_out/apply_r5.log 2>&1
  python -c "
import json
for l in open('gpurun_out/apply_r5.log'):
    d=json.loads(l); print(d['config'], d['b'], round(d['ms_per_apply']*1000,1), {k:v['us'] for k,v in d['passes'].items()})
"
done
BNF_Z_UNROLL=2 timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_r5u2.log 2>&1; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_r5u2.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kpoints_per_s'], d['roofline']['kernel'], d['roofline']['frac']); print({k:v for k,v in d['kernel_ms'].items() if v>1})"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_case.py --quick > gpurun_out/memcheck_r5.log 2>&1; echo memcheck rc=$?
tail -8 gpurun_out/memcheck_r5.log
