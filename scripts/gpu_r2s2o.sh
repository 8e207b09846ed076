# full band paths of configs 1-5 (library defaults: block 4 / guard 4, warm start) after the session-2 kernel changes
timeout 1500 python scripts/path_bench.py --configs 1,2,3,4,5 --out gpurun_out/paths_r02s2.json > gpurun_out/paths_r02s2.log 2>&1; echo paths rc=$?
python -c "
import json; d=json.load(open('gpurun_out/paths_r02s2.json'))
for r in d: print(r['config'], 'kpts/s %.3f' % r['kpoints_per_s'], 'mv/k %.0f' % r['matvecs_per_kpoint'], 'res %.2e' % r['max_residual'], 'golden', r['golden_kpoints'], r['max_rel_dev_vs_oracle'], r['status'], r['failed_kpoints'])"
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r02s2o.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_r02s2o.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','kpoints_per_s','middle','clocks')}, d['roofline']['kernel'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'], d['golden_check'])"
