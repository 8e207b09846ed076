set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
BNF_NO_PLANE=1 BNF_L2_SLABS=1 timeout 900 python -m pytest tests -m gpu -x -q -k "apply_vs or graph or full_size_eigenvalues or config1" > gpurun_out/pytest_slab.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_slab.log
for cfg in "BNF_X=0" "BNF_NO_PLANE=1" "BNF_NO_PLANE=1 BNF_L2_SLABS=1"; do
  echo "== $cfg"
  env $cfg timeout 300 python scripts/bench_apply.py --configs 3,4 --b 2 | cut -c1-400
done
timeout 600 python scripts/sweep_solver.py --config 4 --kidx 5,12 --settings 1:2,2:2,2:4,4:2,4:4 2>&1 | tail -12
