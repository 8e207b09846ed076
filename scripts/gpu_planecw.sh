set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "apply or graph" > gpurun_out/pytest_cw.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_cw.log
BNF_PLANE_CW=16 timeout 600 python -m pytest tests -m gpu -x -q -k "apply_vs_matrixfree or apply_256" > gpurun_out/pytest_cw16.log 2>&1; echo pytest16 rc=$?
tail -3 gpurun_out/pytest_cw16.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 2 > gpurun_out/apply_cw32.log 2>&1
BNF_PLANE_CW=16 timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 2 > gpurun_out/apply_cw16.log 2>&1
cut -c1-330 gpurun_out/apply_cw32.log gpurun_out/apply_cw16.log
