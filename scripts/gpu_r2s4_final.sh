# round-2 (session 4) final evidence at the bench defaults (block 1, guard 2, 2 solvers per GPU):
# bench line, smoke, ncu launch list of one k-point solve, --set full of the CG passes (b = 1),
# then the whole -m gpu suite with durations
TAG=${1:-r02s4f}
timeout 1200 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
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
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 24000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_(zfwd2|zadj2|plane)" -s 3000 -c 3 -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu full rc=$?
unset BNF_PLANE BNF_PLANE_L2 BNF_PLANE_SPLIT BNF_PLANE_T
