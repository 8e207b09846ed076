#!/bin/bash
# session 4, last call: compact evidence (scripts/gpu_r2s4d.sh), then the exhaustive -m gpu matrix
bash scripts/gpu_r2s4d.sh r02s4f
rm -f gpurun_out/r02s4e_durations.txt
BNF_TEST_FULL=1 BNF_DURATIONS_FILE=gpurun_out/r02s4e_durations.txt timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02s4e_pytest_full.txt 2>&1; echo pytest full rc=$?
tail -22 gpurun_out/r02s4e_pytest_full.txt
