#!/bin/bash
# session 4, evidence call (compact: ncu outputs are summarised on the box, raw files dropped if large):
# A/B of the warp-local phase-X exchange and the z-pass register budgets (per-kernel CUDA events), bench
# line at the defaults, smoke, ncu launch list of one k-point solve, --set full of the three CG passes
TAG=${1:-r02s4f}
mkdir -p gpurun_out
python scripts/plane_variants.py --config 4 --b 1 --iters 30 --variants l2,l2_noxw,l2_ld3,l2,l2_noxw,z5,z1029,z517,z2053,z2049,z3077,z3073,z5 > gpurun_out/${TAG}_variants_b1.jsonl 2> gpurun_out/${TAG}_err1.txt
python scripts/plane_variants.py --config 4 --b 2 --iters 30 --variants l2,l2_noxw,z5,z3077,z1029 > gpurun_out/${TAG}_variants_b2.jsonl 2> gpurun_out/${TAG}_err2.txt
python scripts/plane_variants.py --config 5 --b 1 --iters 20 --variants l2,l2_split > gpurun_out/${TAG}_variants_c5.jsonl 2> gpurun_out/${TAG}_err3.txt
timeout 1200 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
CMD="python bench.py --steps 1 --warmup 0 --per-gpu 1 --no-e2e --no-cpu"
export BNF_PLANE=1 BNF_PLANE_L2=1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 24000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu launches rc=$?
timeout 900 ncu --set full --clock-control none \
    -k regex:"k_(zfwd2|zadj2|plane)" -s 3000 -c 3 -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu full rc=$?
python scripts/ncu_summary.py --launches gpurun_out/launches_$TAG.csv --rep gpurun_out/full_$TAG.ncu-rep --out gpurun_out/${TAG}; echo summary rc=$?
head -400 gpurun_out/launches_$TAG.csv > gpurun_out/launches_${TAG}_head400.csv
rm -f gpurun_out/launches_$TAG.csv
du -sh gpurun_out; ls -la gpurun_out
[ $(du -sm gpurun_out | cut -f1) -gt 50 ] && rm -f gpurun_out/full_$TAG.ncu-rep
exit 0
