set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r6.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_r6.log
timeout 900 python bench.py > gpurun_out/bench_r6.log 2>&1; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_r6.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kpoints_per_s'], d['roofline']['kernel'], d['roofline']['frac']); print({k:v for k,v in d['kernel_ms'].items() if v>1}); print(d['e2e']); print(d['cpu_baseline']); print(d['clocks'])"
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_r6.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 2500 --csv \
    --log-file gpurun_out/launches_r6.csv $CMD > gpurun_out/ncu_launch_r6.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(zfwd2|zadj2|xpass_fast|ypass_fast|gemm)" -s 60 -c 8 \
    -o gpurun_out/full_r6 $CMD > gpurun_out/ncu_full_r6.log 2>&1
echo ncu rc=$?
