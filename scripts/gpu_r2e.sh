python paper_1806_10284_b200/build.py > gpurun_out/build_r2e.log 2>&1 || { tail -20 gpurun_out/build_r2e.log; exit 1; }
for c in 4 2 5; do timeout 300 python scripts/plane_variants.py --config $c --b 2 --iters 10 --variants l2,tma_shfl,tma; done > gpurun_out/pv_r2e.log 2>&1; echo pv rc=$?
python - <<'PY'
import json
for line in open("gpurun_out/pv_r2e.log"):
    try: d = json.loads(line)
    except Exception: print(line.strip()[:300]); continue
    print(d["variant"], d["config"], "ms/iter %.4f dev %s" % (d["ms_per_iter"], d["dev_vs_first"]), {k: (v["us"], v["frac"]) for k, v in d["passes"].items() if "cg" in k and "finish" not in k})
PY
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_c_abi.py -q -k "tma_shfl and not 256 or dist_single or field_post or kpath_concurrent or c_consumer or block_sizes or graph_cg or warm_start" > gpurun_out/pytest_r2e.log 2>&1; echo pytest rc=$?; tail -8 gpurun_out/pytest_r2e.log
