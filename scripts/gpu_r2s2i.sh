for z in 4 68; do
BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 20 --variants l2 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('zcfg',$z, round(d['ms_per_iter'],4), {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'z' in k})"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "zadj3" --timeout 400 > gpurun_out/pytest_r3i.log 2>&1; echo pytest rc=$?; tail -30 gpurun_out/pytest_r3i.log | grep -v "^  " | tail -12
