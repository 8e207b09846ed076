#!/bin/bash
# Round 2 session 4: (i) phase-X warp-local exchange of the L2 plane pass (default; BNF_PLANE_LD bit 4 restores the CTA barriers), the load
# policies (bits 1, 2) and the z-pass register budgets (BNF_ZCFG bits 9-11) at config 4 (128^3), b = 1, 2:
# per-kernel CUDA events over CG iterations (scripts/plane_variants.py); (ii) parity of the new variant.
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/r02s4a_clk.txt
python scripts/plane_variants.py --config 4 --b 1 --iters 60 --variants l2,l2_noxw,l2_ld1,l2_ld2,l2_ld3,l2_noxw_ld3,l2,l2_noxw > gpurun_out/r02s4a_plane.jsonl 2> gpurun_out/r02s4a_err1.txt
python scripts/plane_variants.py --config 4 --b 1 --iters 60 --variants z5,z1029,z517,z2053,z2049,z3077,z3073,z5 > gpurun_out/r02s4a_zcfg.jsonl 2> gpurun_out/r02s4a_err2.txt
python scripts/plane_variants.py --config 4 --b 2 --iters 30 --variants l2,l2_noxw,l2_ld3,z5,z3077,z1029 > gpurun_out/r02s4a_b2.jsonl 2> gpurun_out/r02s4a_err3.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/r02s4a_clk.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "test_forced_middle_vs_oracle_full_size and (l2 or yxy)" > gpurun_out/r02s4a_pytest_xw.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02s4a_pytest_xw.txt
cat gpurun_out/r02s4a_plane.jsonl | cut -c1-330
