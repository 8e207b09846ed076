# bench: concurrent solvers per GPU x block size at k12+ (kernel-only; e2e + oracle off for speed)
for cfg in "1 1 1" "1 1 2" "2 2 2" "1 1 3" "2 2 1"; do set -- $cfg
timeout 600 python bench.py --block $1 --guard $2 --per-gpu $3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "
import sys,json
l=sys.stdin.read()
try: d=json.loads(l)
except Exception: print(l[-1500:]); sys.exit()
print('block',$1,'guard',$2,'per_gpu',$3,'matvecs/s',round(d['value']),'kpts/s',round(d['kpoints_per_s'],3),'mv/k',d['solver']['matvecs_per_kpoint'],'gold',d['golden_check'], 'res', d['solver']['max_residual'])"
done
