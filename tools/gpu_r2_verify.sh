#!/bin/bash
# full GPU suite + short bench lines (cfg2 / cfg3 / cfg3r2 / cfg5)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for c in cfg2 cfg3 cfg3r2 cfg5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-per-op --no-north-star --no-row-shard 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c us/step %.2f marginal %.2f kernel %.2f frac %.3f' % (1e3*d['ms_per_step'], d.get('us_per_step_marginal') or -1, 1e3*d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
