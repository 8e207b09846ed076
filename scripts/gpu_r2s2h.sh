timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "zadj3" > gpurun_out/pytest_r3h.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r3h.log
for z in 4 36; do
BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('zcfg',$z,'z3', round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'z' in k})"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_zadj3" -c 1 \
  -o gpurun_out/r3h_zadj3 python scripts/plane_variants.py --config 4 --b 2 --iters 2 --variants l2 > gpurun_out/r3h_ncu.log 2>&1; echo ncu rc=$?
