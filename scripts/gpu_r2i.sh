python paper_1806_10284_b200/build.py > gpurun_out/build_r2i.log 2>&1 || { tail -20 gpurun_out/build_r2i.log; exit 1; }
timeout 600 python scripts/path_bench.py --configs 3 --per-gpu 2 --kmax 10 > gpurun_out/pg2_c3_r2i.log 2>&1; echo pg2 rc=$?; grep -E "FAILED|kpoints_per_s" gpurun_out/pg2_c3_r2i.log | cut -c1-400
timeout 600 python scripts/path_bench.py --configs 3 --per-gpu 1 --kmax 10 > gpurun_out/pg1_c3_r2i.log 2>&1; echo pg1 rc=$?; grep -E "FAILED|kpoints_per_s" gpurun_out/pg1_c3_r2i.log | cut -c1-300
timeout 900 python scripts/path_bench.py --configs 4 --kmax 3 --method 1 --guard 4 > gpurun_out/lob_c4_r2i.log 2>&1; echo lob rc=$?; grep -E "FAILED|kpoints_per_s" gpurun_out/lob_c4_r2i.log | cut -c1-600
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "gyroid or large_prime or unsupported_axis or lobpcg" > gpurun_out/pytest_r2i.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_r2i.log
