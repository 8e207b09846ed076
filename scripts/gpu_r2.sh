set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_r2.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 2 | cut -c1-330
BNF_PHASE_PROF=1 timeout 300 python scripts/phase_prof.py --config 4 --b 2
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r2.log 2>&1; echo bench rc=$?
cut -c1-1500 gpurun_out/bench_r2.log
