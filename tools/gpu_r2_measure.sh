cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
for c in jd cfg3r2 cfg3 cfg4; do
  extra="--no-cpu-baseline --no-north-star --no-row-shard"; [ "$c" = cfg4 ] && extra="$extra --no-per-op --steps 20"
  timeout 900 python bench.py --config $c $extra > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 300 --csv --log-file gpurun_out/r2_launches_bench_cfg2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-per-op --no-north-star --no-row-shard > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ns_sweep -s 3 -c 1 -o gpurun_out/r2_prof_ns_sweep python tools/prof_eval.py --config ns2000 --mask ns --reps 6 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pick_update -s 5 -c 1 -o gpurun_out/r2_prof_pick_cfg2 python tools/prof_dev.py --config cfg2 > /dev/null 2>&1
python - <<'PY'
import json
for c in ["default","jd","cfg3r2","cfg3","cfg4","reference"]:
    try:
        d=json.loads(open(f"gpurun_out/r2_bench_{c}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(c, "FAILED", e); continue
    r=d.get("roofline") or {}
    print(c, "value %.4g"%d["value"], "us/step %.2f"%(1e3*d["ms_per_step"]), "frac %.3f"%r.get("frac",0), "kernel_us %.2f"%(1e3*r.get("kernel_ms",0)), "clk", (d.get("clocks") or {}).get("sm_mhz"))
    for k,v in (d.get("per_operator_steady_state") or {}).items(): print("   ",k, "%.2f us"%v["us_per_sweep"])
    if "north_star" in d: print("   NS", {k: d["north_star"][k] for k in ("us_per_sweep","kernel_us","alu_frac_kernel","alu_frac_sweep","hbm_frac_sweep")})
PY
