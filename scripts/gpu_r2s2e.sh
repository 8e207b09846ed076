# bench block / guard sweep at the bench k-points (k12-15), kernel-only and e2e off for speed
for bg in "1 1" "1 2" "2 2" "3 2"; do set -- $bg
timeout 600 python bench.py --block $1 --guard $2 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('block',$1,'guard',$2,'matvecs/s',round(d['value']),'kpts/s',round(d['kpoints_per_s'],3),'mv/k',d['solver']['matvecs_per_kpoint'],'plane us',round(d['roofline']['avg_launch_us'],1), d['roofline']['kernel'])"
done
