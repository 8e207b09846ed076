# z-pass register-prefetch rework: A/B of BNF_ZCFG values, z-variant parity
python paper_1806_10284_b200/build.py > gpurun_out/build_r2j.log 2>&1 || { tail -20 gpurun_out/build_r2j.log; exit 1; }
for z in 4 0 12 8 1; do
  BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 30 --variants tma_shfl,l2 2>&1 | sed "s/^/zcfg=$z /" >> gpurun_out/zcfg_r2j.log
done
grep -o 'zcfg=[0-9]* {"variant": "[a-z_]*"\|"z[a-z0-9_]*": {"us": [0-9.]*' gpurun_out/zcfg_r2j.log | paste -sd' ' | sed 's/zcfg=/\nzcfg=/g'
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "zpass_variants or cg_fused_iterations or graph_cg_equals_eager" > gpurun_out/pytest_r2j.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_r2j.log
timeout 600 python scripts/path_bench.py --configs 3 --per-gpu 2 --kmax 10 > gpurun_out/pg2_c3_r2j.log 2>&1; echo pg2 rc=$?; grep -E "FAILED|kpoints_per_s" gpurun_out/pg2_c3_r2j.log | cut -c1-300
timeout 600 python scripts/path_bench.py --configs 2,3 --per-gpu 3 --kmax 12 > gpurun_out/pg3_r2j.log 2>&1; echo pg3 rc=$?; grep -E "FAILED|kpoints_per_s" gpurun_out/pg3_r2j.log | cut -c1-300
