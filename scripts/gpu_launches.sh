# ncu launch list over one whole bench step (the timed k-point solve), for the
# per-kernel share of the step; the bench-selected real-space middle is forced
TAG=${1:-launches}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 || exit 1
MIDDLE=$(python -c "import json; print(json.loads(open('gpurun_out/prof_plain_$TAG.log').read().strip().splitlines()[-1])['middle'])")
case "$MIDDLE" in
  plane_l2) export BNF_PLANE=1 BNF_PLANE_L2=1 ;;
  plane_cluster) export BNF_PLANE=1 ;;
  *) export BNF_NO_PLANE=1 ;;
esac
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 14000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo ncu rc=$?
