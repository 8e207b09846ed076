# round-2 evidence: band paths (per-GPU concurrency, relaxed inner CG), apply micro-bench, oracle per config,
# launch list of one bench step, ncu --set full of the CG passes
TAG=${1:-r02}
python paper_1806_10284_b200/build.py > gpurun_out/build_ev_$TAG.log 2>&1 || exit 1
timeout 900 python scripts/path_bench.py --configs 1,2,3,4,5 --out gpurun_out/paths_$TAG.json > gpurun_out/paths_$TAG.log 2>&1; echo paths rc=$?
timeout 600 python scripts/path_bench.py --configs 2,3 --per-gpu 2 --out gpurun_out/paths_pg2_$TAG.json > gpurun_out/paths_pg2_$TAG.log 2>&1; echo paths pg2 rc=$?
timeout 600 python scripts/path_bench.py --configs 2 --per-gpu 3 --out gpurun_out/paths_pg3_$TAG.json > gpurun_out/paths_pg3_$TAG.log 2>&1; echo paths pg3 rc=$?
timeout 900 python scripts/path_bench.py --configs 2,4 --kmax 6 --relax-inner 1 --out gpurun_out/paths_relax_$TAG.json > gpurun_out/paths_relax_$TAG.log 2>&1; echo paths relax rc=$?
timeout 900 python scripts/path_bench.py --configs 2,4 --kmax 6 --method 1 --guard 4 --out gpurun_out/paths_lobpcg_$TAG.json > gpurun_out/paths_lobpcg_$TAG.log 2>&1; echo paths lobpcg rc=$?
BNF_GEMM_V2=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_gemmv2_$TAG.log 2>&1; echo gemmv2 rc=$?
timeout 600 python scripts/bench_apply.py --configs 2,3,4,5 --b 1,2 > gpurun_out/apply_$TAG.log 2>&1; echo apply rc=$?
for c in 2 3 4 5; do timeout 300 python bench.py --impl reference --steps 1 --warmup 0 --config $c; done > gpurun_out/oracle_$TAG.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 4000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(zfwd2|zadj2|plane|gemm)" -s 3000 -c 6 \
    -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu rc=$?
for f in paths_$TAG paths_pg2_$TAG paths_pg3_$TAG paths_relax_$TAG paths_lobpcg_$TAG; do python -c "
import json; d=json.load(open('gpurun_out/$f.json'))
for r in d: print('$f', r['config'], 'kpts/s %.3f' % r['kpoints_per_s'], 'mv/k %.0f' % r['matvecs_per_kpoint'], 'res %.2e' % r['max_residual'], 'golden', r['golden_kpoints'], r['max_rel_dev_vs_oracle'])"; done
tail -1 gpurun_out/bench_gemmv2_$TAG.log | cut -c1-400
