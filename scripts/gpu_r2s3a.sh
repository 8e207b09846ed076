#!/bin/bash
# Round 2 session 3: plane-pass load policies (BNF_PLANE_LD) and z-pass register budgets (BNF_ZCFG bits 9-11)
# at config 4 (128^3), b = 1 and b = 2, per-kernel CUDA events over CG iterations (scripts/plane_variants.py).
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/r02s3a_clk.txt
python scripts/plane_variants.py --config 4 --b 1 --iters 60 --variants l2,l2_ld1,l2_ld2,l2_ld3,l2,l2_ld3 > gpurun_out/r02s3a_plane_ld.jsonl 2> gpurun_out/r02s3a_err1.txt
python scripts/plane_variants.py --config 4 --b 1 --iters 60 --variants z5,z1029,z517,z2053,z2049,z3077,z3073,z5 > gpurun_out/r02s3a_zcfg.jsonl 2> gpurun_out/r02s3a_err2.txt
python scripts/plane_variants.py --config 4 --b 2 --iters 30 --variants l2,l2_ld3,z5,z3077,z1029 > gpurun_out/r02s3a_b2.jsonl 2> gpurun_out/r02s3a_err3.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/r02s3a_clk.txt
