# part 2 of the session-2 evidence: the forced-variant test families
TAG=${1:-r02s2f}
timeout 3300 python -m pytest tests/test_gpu_parity.py -m gpu -q --durations=20 -k "test_forced_middle_vs_oracle_full_size or test_cg_fused_iterations_elementwise or zadj3" > gpurun_out/pytest2_$TAG.log 2>&1; echo pytest2 rc=$?
tail -26 gpurun_out/pytest2_$TAG.log
