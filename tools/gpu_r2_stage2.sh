#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu -x -k "device or lockstep or slack or step or relayout or pd or reversed" 2>&1 | tail -2
for c in cfg2 cfg3r2 cfg4; do python tools/probe_step.py --config $c --steps 6 2>&1 | tail -3 | cut -c1-400; done
python tools/step_times.py --config cfg3r2 --steps 120 --show 60
for c in cfg2 cfg3r2 cfg3; do for K in 20 60; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-per-op --no-north-star --no-row-shard --steps $K 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c K=$K us/step %.2f marginal %.2f' % (1e3*d['ms_per_step'], d.get('us_per_step_marginal') or -1))"
done; done
