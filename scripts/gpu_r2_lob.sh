python paper_1806_10284_b200/build.py > gpurun_out/build_lob.log 2>&1 || { tail -20 gpurun_out/build_lob.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "lobpcg or relaxed or field_post" > gpurun_out/pytest_lob.log 2>&1; echo pytest rc=$?; tail -6 gpurun_out/pytest_lob.log
for args in "--method 0" "--method 1 --guard 4" "--method 0 --relax-inner 1"; do
  timeout 900 python scripts/path_bench.py --configs 2,4 --kmax 4 $args 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('$args', d['config'], 'kpts/s %.3f' % d['kpoints_per_s'], 'mv/k %.0f' % d['matvecs_per_kpoint'], 'res %.2e' % d['max_residual'], 'golden', d['golden_kpoints'], d['max_rel_dev_vs_oracle'])"
done
