# plane options (stage roots in smem, even/odd x phase with 256-bit accesses) and the alpha fold:
# timing at 128^3 (b = 1, 2), then parity of the new code paths
for b in 1 2; do
for v in l2 l2_rs l2_xeo l2_xeo_rs; do
timeout 300 python scripts/plane_variants.py --config 4 --b $b --iters 20 --variants $v 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('b',$b,'$v', round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if k not in ('copy','dot','dot_final','cg_init','cg_xfinal')})"
done; done
BNF_NO_ALPHA_FOLD=1 timeout 300 python scripts/plane_variants.py --config 4 --b 1 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('nofold b1 l2', round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if k not in ('copy','dot','dot_final','cg_init','cg_xfinal')})"
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "l2_rs or l2_xeo or graph_cg_equals_eager or cg_solve_converges or block_sizes or full_size_eigenvalues_vs_oracle" > gpurun_out/pytest_r2s2m.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2s2m.log
