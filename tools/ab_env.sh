#!/bin/bash
# A/B step times of one build under environment variants: bash tools/ab_env.sh "cfg2 cfg4" "" "TGA_X=1" ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFGS=$1; shift
for rep in 1 2 3; do
  for envs in "$@"; do
    for c in $CFGS; do
      env $envs timeout 600 python bench.py --config $c --no-cpu-baseline --no-per-op --no-north-star --no-row-shard 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%-22s $c us/step %.2f marginal %.2f kernel %.2f' % ('[$envs]', 1e3*d['ms_per_step'], d.get('us_per_step_marginal') or -1, 1e3*d['roofline']['kernel_ms']))"
    done
  done
done
