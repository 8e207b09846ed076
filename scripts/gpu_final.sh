# end-of-round evidence: all GPU tests, smoke, bench (default), full band paths of all configs,
# apply micro-bench, oracle timings per config, launch list + ncu full of the operator passes
# (the ncu runs force the real-space middle the timed bench selected, since the autotune's
# timing is perturbed under the profiler)
TAG=${1:-final}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
MIDDLE=$(python -c "import json; print(json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1])['middle'])")
case "$MIDDLE" in
  plane_l2) export BNF_PLANE=1 BNF_PLANE_L2=1 ;;
  plane_cluster) export BNF_PLANE=1 ;;
  *) export BNF_NO_PLANE=1 ;;
esac
timeout 1500 python scripts/path_bench.py --configs 1,2,3,4,5 --out gpurun_out/paths_$TAG.json > gpurun_out/paths_$TAG.log 2>&1; echo paths rc=$?
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 1,2 > gpurun_out/apply_$TAG.log 2>&1; echo apply rc=$?
for c in 2 3 4 5; do timeout 300 python bench.py --impl reference --steps 1 --warmup 0 --config $c; done > gpurun_out/oracle_$TAG.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 3000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(zfwd2|zadj2|xpass_fast|ypass_fast|plane)" -s 3000 -c 6 \
    -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu rc=$?
