# concurrent solvers per GPU at 128^3 (config 4)
for pg in 1 2; do
timeout 600 python scripts/path_bench.py --configs 4 --kmax 6 --block 2 --guard 2 --per-gpu $pg 2>&1 | tail -1 | cut -c1-330
done
timeout 600 python scripts/path_bench.py --configs 4 --kmax 6 --block 1 --guard 2 --per-gpu 2 2>&1 | tail -1 | cut -c1-330
timeout 600 python scripts/path_bench.py --configs 4 --kmax 6 --block 2 --guard 2 --per-gpu 3 2>&1 | tail -1 | cut -c1-330
