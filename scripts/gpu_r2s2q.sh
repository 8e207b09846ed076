# alpha partials copied with the U tile (cp.async) vs the old direct-load prologue: timing, then parity
for b in 1 2; do
timeout 300 python scripts/plane_variants.py --config 4 --b $b --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('b',$b, round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if k not in ('copy','dot','dot_final','cg_init','cg_xfinal')})"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "zadj3 or graph_cg_equals_eager or cg_solve_converges or zpass_variants or warm_start or (full_size_eigenvalues_vs_oracle and not c5)" > gpurun_out/pytest_r2s2q.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_r2s2q.log
