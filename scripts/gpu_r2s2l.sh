timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "l2_split" --timeout 600 > gpurun_out/pytest_r2s2l.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2s2l.log
timeout 900 python bench.py > gpurun_out/bench_r2s2l.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_r2s2l.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','kpoints_per_s','middle','gpu_launches','clocks')}, d['roofline'], d['e2e'], d['golden_check'], d['solver'])"
