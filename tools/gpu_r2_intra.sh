cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fields_gpu.py -x -q -k "cfg1 or full_size or lockstep or device or virtual or degenerate" > gpurun_out/pytest_intra.log 2>&1; tail -3 gpurun_out/pytest_intra.log
for env in "" "TGA_INTRA_RIDE=1"; do
  echo "== $env"; env $env python tools/sweep_time.py --config cfg2 --mask all 2>&1 | tail -1
  env $env python tools/sweep_time.py --config cfg2 --mask inter 2>&1 | tail -1
  env $env timeout 600 python bench.py --no-cpu-baseline --no-per-op --no-north-star --no-row-shard --steps 60 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench cfg2 us/step %.2f kernel_us %.2f frac %.3f' % (1e3*d['ms_per_step'], 1e3*d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
