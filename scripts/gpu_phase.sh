set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
BNF_PHASE_PROF=1 timeout 300 python scripts/phase_prof.py --config 4 --b 2 > gpurun_out/phase_c4.log 2>&1
BNF_PHASE_PROF=1 timeout 300 python scripts/phase_prof.py --config 2 --b 2 >> gpurun_out/phase_c4.log 2>&1
BNF_PHASE_PROF=1 timeout 300 python scripts/phase_prof.py --config 5 --b 1 >> gpurun_out/phase_c4.log 2>&1
cat gpurun_out/phase_c4.log
