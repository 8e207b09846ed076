# full check: build, all GPU tests, smoke, bench (+ apply bench)
TAG=${1:-b}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
cat gpurun_out/smoke_$TAG.log | tail -2
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
cut -c1-3000 gpurun_out/bench_$TAG.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 1,2 > gpurun_out/apply_$TAG.log 2>&1; echo apply rc=$?
cut -c1-400 gpurun_out/apply_$TAG.log
