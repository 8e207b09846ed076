set -x
python paper_1806_10284_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
export BNF_NO_PLANE=1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_cg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_xpass_fast|k_zadj2|k_gemm_tn" -s 200 -c 6 \
    -o gpurun_out/full_cg2 $CMD > gpurun_out/ncu_full_cg2.log 2>&1
echo ncu rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/prof_plain_cg2.log').read().strip().splitlines()[-1])
print(d['value'], d['kernel_ms'])"
