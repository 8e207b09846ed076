# L2 plane pass split over a 2-CTA cluster per plane (BNF_PLANE_SPLIT=2) vs one CTA per plane
for b in 1 2; do for sp in 1 2; do
BNF_PLANE_SPLIT=$sp timeout 300 python scripts/plane_variants.py --config 4 --b $b --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('b',$b,'split',$sp, round(d['ms_per_iter'],4), d['dev_vs_first'], {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'plane' in k})"
done; done
for c in 2 5; do for sp in 1 2; do
BNF_PLANE_SPLIT=$sp timeout 300 python scripts/plane_variants.py --config $c --b 2 --iters 10 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('cfg',$c,'split',$sp, round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'plane' in k})"
done; done
