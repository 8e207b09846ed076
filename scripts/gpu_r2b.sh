python paper_1806_10284_b200/build.py > gpurun_out/build_r2b.log 2>&1 || { tail -20 gpurun_out/build_r2b.log; exit 1; }
( cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o xchg xchg.cu && ./xchg ) > gpurun_out/micro_xchg.log 2>&1; cat gpurun_out/micro_xchg.log
timeout 600 python scripts/plane_variants.py --config 4 --b 2 --iters 10 > gpurun_out/plane_variants_r2b.log 2>&1; echo pv rc=$?; cut -c1-600 gpurun_out/plane_variants_r2b.log
PYTEST_ARGS="-x" bash scripts/gpu_check.sh r2b
