# build -> operator parity -> eigen parity (full-size, fast path) -> apply bench -> ncu of the passes
TAG=${1:-it}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "apply or batch or full_size or config1 or solve_deter" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_$TAG.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 1,2 > gpurun_out/apply_$TAG.log 2>&1; echo apply rc=$?
cut -c1-600 gpurun_out/apply_$TAG.log
timeout 300 python scripts/bench_apply.py --configs 4 --b 1 --reps 2 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_plane|k_zfwd2|k_zadj2" -c 3 \
    -o gpurun_out/full_$TAG python scripts/bench_apply.py --configs 4 --b 1 --reps 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc=$?
