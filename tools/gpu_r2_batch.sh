cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1

timeout 900 python bench.py --config cfg5 --no-cpu-baseline --steps 20 2>/dev/null > gpurun_out/r2_bench_cfg5.json; python -c "import json; d=json.loads(open('gpurun_out/r2_bench_cfg5.json').read().strip().splitlines()[-1]); print('cfg5 ms/step %.3f kernel_ms %.3f frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
timeout 900 python bench.py --config cfg4 --no-cpu-baseline --no-per-op --no-north-star --no-row-shard --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 us/step %.2f kernel_us %.2f' % (1e3*d['ms_per_step'], 1e3*d['roofline']['kernel_ms']))"
timeout 900 ncu --set full --clock-control none -k regex:k_inter_fast_batch -s 2 -c 1 -o gpurun_out/r2_prof_batch python tools/prof_batch.py > /dev/null 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
