cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "cfg4 or full_size or device_resident or slack or virtual" 2>&1 | tail -2
for c in cfg4 cfg2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-north-star --no-row-shard --no-per-op --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c us/step %.2f kernel_us %.2f frac %.3f' % (1e3*d['ms_per_step'], 1e3*d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
git -C $GRAFT_REPO_ROOT log --oneline -1 2>/dev/null
