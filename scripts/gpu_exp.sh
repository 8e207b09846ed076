set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "apply_vs_matrixfree or graph or full_size_eigenvalues or config1" > gpurun_out/pytest_exp.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_exp.log
BNF_PLANE_CW=64 timeout 600 python -m pytest tests -m gpu -x -q -k "apply_vs_matrixfree" > gpurun_out/pytest_exp64.log 2>&1; echo pytest64 rc=$?
tail -2 gpurun_out/pytest_exp64.log
timeout 300 python scripts/bench_apply.py --configs 4,5 --b 2 > gpurun_out/apply_exp.log 2>&1
BNF_PLANE_CW=64 timeout 300 python scripts/bench_apply.py --configs 4 --b 2 > gpurun_out/apply_exp64.log 2>&1
cut -c1-330 gpurun_out/apply_exp.log gpurun_out/apply_exp64.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_exp.log 2>&1; echo bench rc=$?
cut -c1-2500 gpurun_out/bench_exp.log
