# paired-plane TMA variant (plane_t 3): parity, then timing vs the other middles
python paper_1806_10284_b200/build.py > gpurun_out/build_r2k.log 2>&1 || { tail -20 gpurun_out/build_r2k.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_pair" > gpurun_out/pytest_r2k.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_r2k.log
for c in 4 2 5; do
  timeout 300 python scripts/plane_variants.py --config $c --b 2 --iters 20 --variants tma_shfl,tma_pair,l2 2>&1 | tee -a gpurun_out/pair_r2k.log | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['variant'], d['config'], round(d['ms_per_iter'],4), d['dev_vs_first'], {k:(v['us'],v['frac']) for k,v in d['passes'].items() if 'plane' in k})
"
done
