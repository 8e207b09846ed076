# round-2 validation: every -m gpu test, smoke, default bench (profiles/r02_*)
TAG=${1:-r02}
python paper_1806_10284_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -12 gpurun_out/pytest_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-3000
