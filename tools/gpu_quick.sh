#!/bin/bash
# Quick GPU iteration: parity tests, bench lines, optional ncu capture of one kernel.
#   KERNEL=<regex> CONFIG=<cfg> to capture; BENCHES="cfg2 ns2000" to choose bench configs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { cat gpurun_out/smoke.log; exit 1; }
if [ -z "$NOTEST" ]; then timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; fi
for c in ${BENCHES:-cfg2 ns2000}; do
  extra="--no-cpu-baseline"; [ "$c" = cfg4 ] && extra="$extra --no-per-op --steps 20 --warmup 3"
  timeout 600 python bench.py --config $c $extra > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", open(f"gpurun_out/bench_{c}.err").read()[-2000:]); sys.exit()
r=d.get("roofline") or {}
print(c, "value %.4g"%d["value"], "us/step %.2f"%(1e3*d["ms_per_step"]), "inter_us %.2f"%(1e3*r.get("kernel_ms",0)), "frac %.3f"%r.get("frac",0), "clk", d.get("clocks"))
for k,v in (d.get("per_operator_steady_state") or {}).items(): print("   ",k, "%.2f us"%v["us_per_sweep"])
PY
done
if [ -n "$KERNEL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KERNEL -s ${SKIP:-4} -c 1 -o gpurun_out/prof_${TAG:-x} python tools/prof_dev.py --config ${CONFIG:-cfg2} --steps 6 > gpurun_out/prof_${TAG:-x}.log 2>&1
  tail -2 gpurun_out/prof_${TAG:-x}.log
fi
if [ -n "$KERNEL2" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KERNEL2 -s ${SKIP:-4} -c 1 -o gpurun_out/prof_${TAG2:-y} python tools/prof_dev.py --config ${CONFIG2:-cfg2} --steps 6 > gpurun_out/prof_${TAG2:-y}.log 2>&1
  tail -2 gpurun_out/prof_${TAG2:-y}.log
fi
