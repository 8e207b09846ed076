# ncu full captures of the Lanczos block kernels (X^*Y partial products,
# W -= V C) at the bench workload; SKIP = matching launches skipped first
# (larger SKIP = later Lanczos steps, wider basis)
TAG=${1:-gemm}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_gemm_(tn_partial|nn)" -s ${SKIP:-60} -c 6 \
    -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu rc=$?
