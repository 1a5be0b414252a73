#!/bin/bash
# pick/update latency iteration: build, device-step parity tests, phase probe, cfg2/cfg3r2/cfg4 step times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x -k "${PYTEST_K:-device or lockstep or slack or descent or step}" 2>&1 | tail -2
python tools/probe_step.py --config cfg2 --steps 14 2>&1 | tail -1
for c in ${CONFIGS:-cfg2 cfg3r2 cfg4}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-per-op --no-north-star --no-row-shard 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c us/step %.2f marginal %.2f kernel %.2f frac %.3f' % (1e3*d['ms_per_step'], d.get('us_per_step_marginal') or -1, 1e3*d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
