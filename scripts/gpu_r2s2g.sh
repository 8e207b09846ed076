# zadj3 (TMA-pipelined adjoint z pass): parity vs zadj2 + timing
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "zadj3" > gpurun_out/pytest_r3g.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_r3g.log
for z in 4 36; do
BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('zcfg',$z,'z3', round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'z' in k})"
done
BNF_NO_Z3=1 timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('z2', round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'z' in k})"
