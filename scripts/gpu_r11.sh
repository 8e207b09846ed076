set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "graph or config1 or full_size_eigenvalues or warm or plane_l2 or deter" > gpurun_out/pytest_r11.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_r11.log
for e in "BNF_X=1" "BNF_CG_EXT_A=1"; do
env $e timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_r11.log 2>&1; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_r11.log').read().strip().splitlines()[-1])
print('$e', d['value'], d['ms_per_step'], d['kpoints_per_s'], d['middle'], d['roofline']['kernel'], d['roofline']['frac']); print({k:v for k,v in d['kernel_ms'].items() if v>1})"
done
