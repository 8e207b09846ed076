for b in 1 2; do for z in 4 5 6 7; do
BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b $b --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('b',$b,'zcfg',$z, round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if k in ('zfwd2_cg','zadj2_cg')})"
done; done
