# build -> fast parity subset -> bench (graph CG) -> apply bench -> ncu of plane (+z) at 128^3
TAG=${1:-it}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "apply or batch or config1 or small_config or degenerate or vacuum or deter or full_size_eigenvalues" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
cut -c1-3500 gpurun_out/bench_$TAG.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 1,2 > gpurun_out/apply_$TAG.log 2>&1; echo apply rc=$?
cut -c1-400 gpurun_out/apply_$TAG.log
timeout 300 python scripts/bench_apply.py --configs 4 --b 2 --reps 2 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_plane|k_zfwd2|k_zadj2" -c 3 \
    -o gpurun_out/full_$TAG python scripts/bench_apply.py --configs 4 --b 2 --reps 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc=$?
