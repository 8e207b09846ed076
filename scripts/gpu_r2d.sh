python paper_1806_10284_b200/build.py > gpurun_out/build_r2d.log 2>&1 || { tail -20 gpurun_out/build_r2d.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma or dist_single" > gpurun_out/pytest_r2d.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_r2d.log
for c in 4 2 5; do timeout 300 python scripts/plane_variants.py --config $c --b 2 --iters 10 --variants l2,tma; done > gpurun_out/pv_r2d.log 2>&1; echo pv rc=$?
python - <<'PY'
import json
for line in open("gpurun_out/pv_r2d.log"):
    try: d = json.loads(line)
    except Exception: print(line.strip()[:300]); continue
    print(d["variant"], d["config"], "ms/iter %.4f dev %s" % (d["ms_per_iter"], d["dev_vs_first"]), {k: (v["us"], v["frac"]) for k, v in d["passes"].items() if "cg" in k and "finish" not in k})
PY
CMD="python scripts/plane_variants.py --config 4 --b 2 --iters 4 --variants tma"
$CMD > gpurun_out/ncu_plain_r2d.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_plane_t|k_zadj2|k_zfwd2" -s 9 -c 3 -o gpurun_out/prof_r2d $CMD > gpurun_out/ncu_r2d.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_r2d.log
