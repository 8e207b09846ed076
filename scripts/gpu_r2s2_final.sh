# round-2 (session 2) evidence at the bench defaults (block 1, guard 2, 2 solvers per GPU):
# every -m gpu test, smoke, the bench line, an ncu launch list of one k-point solve and a
# --set full capture of the three CG passes (b = 1)
TAG=${1:-r02s2}
python paper_1806_10284_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
timeout 1200 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-600
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
CMD="python bench.py --steps 1 --warmup 0 --per-gpu 1 --no-e2e --no-cpu"
MIDDLE=$(python -c "import json; print(json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1])['middle'])")
case "$MIDDLE" in
  plane_l2) export BNF_PLANE=1 BNF_PLANE_L2=1 ;;
  plane_l2s) export BNF_PLANE=1 BNF_PLANE_L2=1 BNF_PLANE_SPLIT=2 ;;
  plane_ts) export BNF_PLANE_T=2 ;;
  plane_tp) export BNF_PLANE_T=3 ;;
  *) ;;
esac
echo middle=$MIDDLE
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 24000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_(zfwd2|zadj2|plane)" -s 3000 -c 3 -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu full rc=$?
unset BNF_PLANE BNF_PLANE_L2 BNF_PLANE_SPLIT BNF_PLANE_T
timeout 3300 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_$TAG.log
