set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r10.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_r10.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r10.log 2>&1; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_r10.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kpoints_per_s'], d['middle'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'], d['solver']); print({k:v for k,v in d['kernel_ms'].items() if v>1}); print(d['e2e'])"
