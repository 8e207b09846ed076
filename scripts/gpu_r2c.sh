python paper_1806_10284_b200/build.py > gpurun_out/build_r2c.log 2>&1 || { tail -20 gpurun_out/build_r2c.log; exit 1; }
for z in 0 1 2 3; do BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 4 --b 2 --iters 10 --variants l2 | sed "s/^/zcfg=$z /"; done > gpurun_out/zcfg_r2c.log 2>&1
for z in 0 1 2 3; do BNF_ZCFG=$z timeout 300 python scripts/plane_variants.py --config 2 --b 2 --iters 10 --variants l2 | sed "s/^/zcfg=$z /"; done >> gpurun_out/zcfg_r2c.log 2>&1
python - <<'PY'
import json
for line in open("gpurun_out/zcfg_r2c.log"):
    if not line.startswith("zcfg"): print(line.strip()[:300]); continue
    tag, js = line.split(" ", 1)
    d = json.loads(js)
    print(tag, d["config"], "ms/iter %.4f" % d["ms_per_iter"], {k: (v["us"], v["frac"]) for k, v in d["passes"].items() if "cg" in k and "finish" not in k})
PY
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "virtual_slabs or cg_fused or cg_solve_converges" > gpurun_out/pytest_r2c.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_r2c.log
