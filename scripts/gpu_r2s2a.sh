# round-2 re-entry: current HEAD bench + per-kernel middle timings at 128^3
timeout 900 python bench.py > gpurun_out/bench_r3a.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_r3a.log | cut -c1-2500
timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 20 --variants l2,tma_shfl 2>&1 | tee gpurun_out/pv_r3a.log | cut -c1-600
