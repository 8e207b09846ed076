# source-level ncu of the three CG passes at 128^3, b = 2 (L2 plane forced)
export BNF_PLANE=1 BNF_PLANE_L2=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_plane_l2|k_zadj2|k_zfwd2" -c 3 \
  -o gpurun_out/r3d_passes python scripts/plane_variants.py --config 4 --b 2 --iters 2 --variants l2 > gpurun_out/r3d_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/r3d_ncu.log
