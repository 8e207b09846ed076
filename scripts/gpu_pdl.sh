# A/B of programmatic dependent launch in the CG iteration (BNF_PDL) on the bench workload
set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "pdl or graph or plane_l2 or residual_polish or config1 or deterministic" > gpurun_out/pytest_pdl.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_pdl.log
for pdl in 0 2 1 0 2; do
  BNF_PDL=$pdl timeout 600 python bench.py --no-cpu > gpurun_out/bench_pdl$pdl.log 2>&1
  tail -1 gpurun_out/bench_pdl$pdl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pdl', d['value'], d['e2e']['value'], d['solver']['matvecs_per_kpoint'])"
done
