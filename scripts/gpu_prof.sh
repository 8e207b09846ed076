# ncu evidence for the bench workload (config 4, 128^3, block 2): launch list
# + one full capture of each operator pass.  Usage (under gpurun):
#   bash scripts/gpu_prof.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 3000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(zfwd|zadj|xpass|ypass)_fast" -s 40 -c 5 \
    -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "prof rc=$?"
