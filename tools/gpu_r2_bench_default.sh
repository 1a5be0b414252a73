cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_nccl_gpu.py -x -q > gpurun_out/pytest_nccl.log 2>&1; tail -3 gpurun_out/pytest_nccl.log
( time timeout 900 python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -4 gpurun_out/bench_default.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_default.json").read().strip().splitlines()[-1])
print("value %.4g ms/step %.4f frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["frac"]))
print(json.dumps(d.get("north_star"), indent=0))
print(json.dumps(d.get("row_shard"), indent=0))
PY
