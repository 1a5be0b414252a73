#!/bin/bash
# does the nvidia-smi clock sampler perturb the timed replay?  6 runs each, cfg2 + cfg3r2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for c in cfg2 cfg3r2; do for smi in on off; do for i in 1 2 3 4 5 6; do
  if [ $smi = off ]; then export TGA_BENCH_NO_SMI=1; else unset TGA_BENCH_NO_SMI; fi
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-per-op --no-north-star --no-row-shard 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c smi=$smi us/step %.2f marginal %.2f' % (1e3*d['ms_per_step'], d.get('us_per_step_marginal') or -1))"
done; done; done
