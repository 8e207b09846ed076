python paper_1806_10284_b200/build.py > gpurun_out/build_r2g.log 2>&1 || { tail -20 gpurun_out/build_r2g.log; exit 1; }
CMD="python scripts/plane_variants.py --config 4 --b 2 --iters 3 --variants tma_shfl"
$CMD > gpurun_out/ncu_plain_r2g.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_plane_t|k_zfwd2" -s 6 -c 2 -o gpurun_out/prof_r2g $CMD > gpurun_out/ncu_r2g.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_r2g.log
