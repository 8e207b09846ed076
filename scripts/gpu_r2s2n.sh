# z-pass stage roots + half-angle table in shared memory (default) vs global (BNF_ZCFG bit 256)
for b in 1 2; do for z in 4 260; do
BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b $b --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('b',$b,'zcfg',$z, round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if k not in ('copy','dot','dot_final','cg_init','cg_xfinal')})"
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "zpass_variants or graph_cg_equals_eager or apply_vs_dense" > gpurun_out/pytest_r2s2n.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_r2s2n.log
