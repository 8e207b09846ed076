python paper_1806_10284_b200/build.py > gpurun_out/build_r2h.log 2>&1 || { tail -20 gpurun_out/build_r2h.log; exit 1; }
for z in 0 4 5; do BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 10 --variants l2 | sed "s/^/zcfg=$z /"; done > gpurun_out/pv_r2h.log 2>&1
for z in 0 4; do BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 2 --b 2 --iters 10 --variants l2 | sed "s/^/zcfg=$z /"; done >> gpurun_out/pv_r2h.log 2>&1
for z in 0 4; do BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 5 --b 2 --iters 4 --variants l2 | sed "s/^/zcfg=$z /"; done >> gpurun_out/pv_r2h.log 2>&1
python - <<'PY'
import json
for line in open("gpurun_out/pv_r2h.log"):
    if not line.startswith("zcfg"): print(line.strip()[:300]); continue
    tag, js = line.split(" ", 1)
    d = json.loads(js)
    print(tag, d["variant"], d["config"], "ms/iter %.4f" % d["ms_per_iter"], {k: (v["us"], v["frac"]) for k, v in d["passes"].items() if "cg" in k and "finish" not in k and "init" not in k})
PY
BNF_GEMM_V1=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_gemmv1_r2h.log 2>&1; tail -1 gpurun_out/bench_gemmv1_r2h.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gemm v1', d['value'], d['kpoints_per_s'], {k:v for k,v in d['kernel_ms'].items() if 'gemm' in k})"
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_gemmv2_r2h.log 2>&1; tail -1 gpurun_out/bench_gemmv2_r2h.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gemm v2', d['value'], d['kpoints_per_s'], {k:v for k,v in d['kernel_ms'].items() if 'gemm' in k})"
