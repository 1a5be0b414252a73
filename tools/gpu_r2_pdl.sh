cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_ns_gpu.py tests/test_nccl_gpu.py -q -x 2>&1 | tail -2
for c in ns2000 cfg2 cfg4; do python tools/sweep_time.py --config $c --mask ns | tail -1; done
timeout 900 python bench.py --no-cpu-baseline --no-per-op --no-row-shard --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ns=d['north_star']; print('NS us_per_sweep %.2f kernel_us %.2f alu_sweep %.3f' % (ns['us_per_sweep'], ns['kernel_us'], ns['alu_frac_sweep']))"
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
