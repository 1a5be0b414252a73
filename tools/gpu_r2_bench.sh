#!/bin/bash
# bench lines (BENCHES="cfg2 ns2000 ..."; EXTRA="--score penalised" etc) -> gpurun_out/bench_<tag>.json + summary
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for c in ${BENCHES:-cfg2 ns2000}; do
  tag=${c}${TAG:+_$TAG}
  extra="--no-cpu-baseline $EXTRA"; [ "$c" = cfg4 ] && extra="$extra --no-per-op --steps 20 --warmup 3"
  timeout 900 python bench.py --config $c $extra > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
  python - "$tag" <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", open(f"gpurun_out/bench_{c}.err").read()[-2000:]); sys.exit()
r=d.get("roofline") or {}
print(c, "value %.4g"%d["value"], "us/step %.2f"%(1e3*d["ms_per_step"]), "kernel_us %.2f"%(1e3*r.get("kernel_ms",0)), "frac %.3f"%r.get("frac",0), "clk", (d.get("clocks") or {}).get("sm_mhz"))
for k,v in (d.get("per_operator_steady_state") or {}).items(): print("   ",k, "%.2f us"%v["us_per_sweep"])
for k in ("north_star",):
    if k in d: print("   ", k, json.dumps(d[k]))
PY
done
