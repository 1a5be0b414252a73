cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for spec in "cfg2 20" "cfg3 100" "ns2000 20" "cfg4 20" "cfg3r2 100"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --granular $2 --no-cpu-baseline --steps 40 > gpurun_out/g_$1.json 2> gpurun_out/g_$1.err
  python - "$1" <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/g_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", open(f"gpurun_out/g_{c}.err").read()[-1500:]); sys.exit()
r=d["roofline"]
print(c, "ETGA value %.4g"%d["value"], "us/step %.2f"%(1e3*d["ms_per_step"]), "sweeps/s %.4g"%d["sweeps_per_s"], "cand/step %.4g"%d["candidates_per_step"], "kernel_us %.2f"%(1e3*r["kernel_ms"]), r["bound"], "frac %.3f"%r["frac"])
PY
done
