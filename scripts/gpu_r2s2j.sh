for z in 132 164 4; do
BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('zcfg',$z, round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'z' in k})"
done
BNF_ZCFG=4 timeout 300 python scripts/plane_variants.py --config 4 --b 1 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('b1 zcfg 4', round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'z' in k})"
BNF_NO_Z3=1 timeout 300 python scripts/plane_variants.py --config 4 --b 1 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('b1 z2', round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'z' in k})"
