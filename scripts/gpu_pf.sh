set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "apply_vs or graph or full_size_eigenvalues or config1" > gpurun_out/pytest_pf.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_pf.log
for cfg in "BNF_PLANE_NOPERSIST=1" "BNF_PLANE_STAGGER=0"; do
  echo "== $cfg"
  env $cfg timeout 300 python scripts/bench_apply.py --configs 3,4 --b 2 | cut -c1-330
done
