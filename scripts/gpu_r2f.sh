python paper_1806_10284_b200/build.py > gpurun_out/build_r2f.log 2>&1 || { tail -20 gpurun_out/build_r2f.log; exit 1; }
for z in 0 4; do BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 10 --variants l2,tma_shfl | sed "s/^/zcfg=$z /"; done > gpurun_out/pv_r2f.log 2>&1
python - <<'PY'
import json
for line in open("gpurun_out/pv_r2f.log"):
    if not line.startswith("zcfg"): print(line.strip()[:300]); continue
    tag, js = line.split(" ", 1)
    d = json.loads(js)
    print(tag, d["variant"], d["config"], "ms/iter %.4f" % d["ms_per_iter"], {k: (v["us"], v["frac"]) for k, v in d["passes"].items() if "cg" in k and "finish" not in k and "init" not in k})
PY
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "field_post or (tma_shfl and 128)" > gpurun_out/pytest_r2f.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_r2f.log
