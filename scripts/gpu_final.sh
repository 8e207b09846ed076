# end-of-round evidence: all GPU tests, smoke, bench (default), launch list + ncu full of the
# dominant kernels, full band paths of all configs
TAG=${1:-final}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
timeout 1500 python scripts/path_bench.py --configs 1,2,3,4,5 --out gpurun_out/paths_$TAG.json > gpurun_out/paths_$TAG.log 2>&1; echo paths rc=$?
cut -c1-300 gpurun_out/paths_$TAG.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 1,2 > gpurun_out/apply_$TAG.log 2>&1; echo apply rc=$?
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 3000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(zfwd2|zadj2|xpass_fast|ypass_fast|plane)" -s 2000 -c 6 \
    -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu rc=$?
