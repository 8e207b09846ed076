#!/bin/bash
# session 4, call C: the core -m gpu matrix with a per-test duration log (survives a killed run)
mkdir -p gpurun_out
rm -f gpurun_out/r02s4c_durations.txt
BNF_DURATIONS_FILE=gpurun_out/r02s4c_durations.txt timeout ${1:-2400} python -m pytest tests -m gpu -q --durations=30 > gpurun_out/r02s4c_pytest.txt 2>&1; echo pytest rc=$?
tail -40 gpurun_out/r02s4c_pytest.txt
