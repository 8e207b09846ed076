set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_cg.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_xpass_fast|k_zadj2|k_ypass_fast|k_zfwd2" -s 40 -c 5 \
    -o gpurun_out/full_cg $CMD > gpurun_out/ncu_full_cg.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu_full_cg.log
