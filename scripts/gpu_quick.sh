# quick GPU check: build, operator parity tests, apply micro-bench, bench
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "apply or batch" > gpurun_out/pytest_apply.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_apply.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 1,2 > gpurun_out/bench_apply.log 2>&1; echo apply rc=$?
cat gpurun_out/bench_apply.log | cut -c1-400
