TAG=${1:-it}
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "apply or graph or full_size_eigenvalues or config1 or small_config" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_$TAG.log
BNF_PHASE_PROF=1 timeout 300 python scripts/phase_prof.py --config 4 --b 2 > gpurun_out/phase_$TAG.log 2>&1
cat gpurun_out/phase_$TAG.log
timeout 300 python scripts/bench_apply.py --configs 2,3,4,5 --b 2 > gpurun_out/apply_$TAG.log 2>&1
cut -c1-330 gpurun_out/apply_$TAG.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
cut -c1-1200 gpurun_out/bench_$TAG.log
