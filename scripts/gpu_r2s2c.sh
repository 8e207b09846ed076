# block-1 solvers, concurrency sweep at 128^3 (config 4), k-points 0-5 and 12-17
for g in 1 2 3; do for pg in 1 2 3; do
timeout 600 python scripts/path_bench.py --configs 4 --kmax 6 --block 1 --guard $g --per-gpu $pg 2>&1 | tail -1 | cut -c1-330
done; done
