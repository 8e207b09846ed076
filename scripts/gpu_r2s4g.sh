#!/bin/bash
# session 4: full band paths of configs 1-5 at the library defaults with the session-4 kernels
# (k-points/s, residual per k, deviation from every oracle golden on the path)
mkdir -p gpurun_out
timeout 1000 python scripts/path_bench.py --configs 1,2,3,4,5 --out gpurun_out/r02s4_paths.json > gpurun_out/r02s4_paths.log 2>&1; echo paths rc=$?
tail -3 gpurun_out/r02s4_paths.log | cut -c1-600
