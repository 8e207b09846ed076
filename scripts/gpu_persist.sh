set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "apply or graph or full_size_eigenvalues or config1 or small_config" > gpurun_out/pytest_p.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_p.log
for cfg in "BNF_PLANE_NOPERSIST=1" "BNF_PLANE_STAGGER=0" "BNF_PLANE_STAGGER=20000" "BNF_PLANE_STAGGER=40000"; do
  echo "== $cfg"
  env $cfg timeout 300 python scripts/bench_apply.py --configs 4,5 --b 2 | cut -c1-330
done
BNF_PLANE_STAGGER=20000 BNF_PHASE_PROF=1 timeout 300 python scripts/phase_prof.py --config 4 --b 2
